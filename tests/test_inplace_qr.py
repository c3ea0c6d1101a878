"""In-place QR host logic (CPU only).

libqrt runs a QR on a single-buffer state (34 qubits on 2 GPUs: 2 x 128 GiB
would not fit) as local bit-transposition passes followed by a pairwise
exchange of slot classes between PEs (csrc/qrt_reorder.cu execute_inplace,
SURVEY.md §7 / §8e).  These tests take the decomposition libqrt computes
(qrt_reorder_inplace_plan) for the reorder maps the host layer really emits
(physical_reorder_plan of scheduler QR events), replay the two kernels' index
logic in numpy — including which PE of a pair handles which half of the
class — and require:
  * every amplitude is read/written by exactly one thread (no race, no gap);
  * the result equals the push exchange's mapping (qrt_reorder_plan) and the
    oracle's perform_qr (dist_sim.cpp:203-240) bit for bit.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import cpu


def bit(x, b):
    return (x >> np.uint64(b)) & np.uint64(1)


def apply_local_pass(sub, pairs, nl):
    """local_swap_kernel: element o swaps with o' (each pair's bits exchanged);
    the lower offset of the two does it."""
    if not pairs:
        return
    o = np.arange(1 << nl, dtype=np.uint64)
    op = o.copy()
    for a, c in pairs:
        ba, bc = bit(o, a), bit(o, c)
        op = op & ~((np.uint64(1) << np.uint64(a)) | (np.uint64(1) << np.uint64(c)))
        op |= (bc << np.uint64(a)) | (ba << np.uint64(c))
    h = op > o
    for pe in range(sub.shape[0]):
        x = sub[pe, o[h]].copy()
        sub[pe, o[h]] = sub[pe, op[h]]
        sub[pe, op[h]] = x


def apply_exchange(sub, cross, nl, p):
    """exchange_kernel: PE j's class s (slot bits d_i = s_i) swaps with PE s's
    class j; the pair's lower PE handles the half with bit f = 0."""
    if not cross:
        return np.ones(sub.shape, dtype=np.int64)
    k = len(cross)
    d = [c[0] for c in cross]
    pb = [c[1] for c in cross]
    used = set(d)
    f = max((x for x in range(nl) if x not in used), default=-1)
    touched = np.zeros(sub.shape, dtype=np.int64)
    o = np.arange(1 << nl, dtype=np.uint64)
    cls = np.zeros(o.shape, dtype=np.int64)
    for i in range(k):
        cls |= bit(o, d[i]).astype(np.int64) << i
    old = sub.copy()
    for j in range(p):
        jc = sum(((j >> pb[i]) & 1) << i for i in range(k))
        for s in range(1 << k):
            if s == jc:
                continue
            sp = j
            for i in range(k):
                sp = (sp & ~(1 << pb[i])) | (((s >> i) & 1) << pb[i])
            sel = cls == s
            if f >= 0:
                sel &= bit(o, f) == np.uint64(0 if j < sp else 1)
            elif j > sp:
                continue
            mine = o[sel]
            partner = mine.copy()
            for i in range(k):
                partner = (partner & ~(np.uint64(1) << np.uint64(d[i]))) | (np.uint64((jc >> i) & 1) << np.uint64(d[i]))
            sub[j, mine] = old[sp, partner]
            sub[sp, partner] = old[j, mine]
            touched[j, mine] += 1
            touched[sp, partner] += 1
    # elements of the staying class are never touched; the rest exactly once
    return touched


def events(qb, n, p, sched):
    c = qb.gen_gatefabric(n, 2 * n, 1, False) if sched != "hea" else qb.gen_hea(n, 4, 1, False)
    d = qb.build_dependency_graph(c)
    fn = qb.adhoc_schedule if sched == "adhoc" else qb.flat_tiling
    return fn(c, d, qb.ClusterShape.flat(p)).qr_events


def push_map(qb, n, p, dest):
    lib = qb.load_libqrt()
    per = 1 << (n - (p.bit_length() - 1))
    out = []
    for pe in range(p):
        dpe = np.zeros(per, dtype=np.uint64)
        doff = np.zeros(per, dtype=np.uint64)
        rel = C.c_uint64()
        assert lib.qrt_reorder_plan(n, p, (C.c_int * n)(*dest), pe, dpe.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    doff.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(rel)) == 0
        out.append((dpe, doff))
    return out


@pytest.mark.parametrize("n,p,sched", [(10, 2, "flat"), (10, 4, "flat"), (12, 8, "flat"), (10, 4, "adhoc"),
                                       (12, 8, "adhoc"), (9, 2, "hea"), (11, 8, "hea"), (6, 4, "adhoc")])
def test_inplace_replay_matches_push_and_oracle(qb, n, p, sched):
    nl = n - (p.bit_length() - 1)
    rng = np.random.default_rng(n * 100 + p)
    phys = list(range(n))
    olay = cpu.Layout(n, p)
    psi = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex128)
    sub = psi.reshape(p, -1).copy()
    want = sub.copy()
    evs = events(qb, n, p, sched)
    assert len(evs) > 0
    for ev in evs[:12]:
        dest, phys_new = qb.physical_reorder_plan(ev, phys)
        l0, l1, cross = qb.inplace_reorder_plan(n, p, dest)
        # push mapping of the same dest, applied out of place
        before = sub.copy()
        expect = np.empty_like(sub)
        for pe, (dpe, doff) in enumerate(push_map(qb, n, p, dest)):
            expect[dpe.astype(np.int64), doff.astype(np.int64)] = before[pe]
        apply_local_pass(sub, l0, nl)
        apply_local_pass(sub, l1, nl)
        touched = apply_exchange(sub, cross, nl, p)
        assert touched.max() <= 1, "an amplitude was swapped twice"
        assert np.array_equal(sub, expect)
        # the oracle's logical perform_qr on the canonical order
        cpu.perform_qr(want, olay.dest_for(ev.after.pos_of))
        olay.adopt(ev.after.pos_of)
        phys = list(phys_new)
        # physical -> logical: compare flattened canonical vectors
        got_canon = cpu.flatten(sub, _qubit_at(phys, n))
        want_canon = cpu.flatten(want, olay.qubit_at)
        assert np.array_equal(got_canon, want_canon)


def _qubit_at(phys, n):
    at = [0] * n
    for q, pos in enumerate(phys):
        at[pos] = q
    return at


def test_relocation_touches_exactly_the_moved_amplitudes(qb):
    """k local<->global pairs: the exchange touches (1 - 2^-k) of every PE —
    qr_data_volume(k, n) amplitudes in total (layout.cpp:91-94)."""
    n, p = 10, 8
    nl = n - 3
    lay = qb.QubitLayout.identity(n, qb.ClusterShape.flat(p))
    for k in (1, 2, 3):
        locals_ = ((1 << nl) - 1) & ~(((1 << k) - 1) << (nl - k)) | (((1 << k) - 1) << nl)
        ev = qb.make_qr_event(lay, locals_)
        dest, _ = qb.physical_reorder_plan(ev, list(range(n)))
        l0, l1, cross = qb.inplace_reorder_plan(n, p, dest)
        assert len(cross) == k and not l0 and not l1
        sub = np.zeros((p, 1 << nl), dtype=np.complex128)
        touched = apply_exchange(sub, cross, nl, p)
        assert int(touched.sum()) == qb.qr_data_volume(k, n)


def test_refill_is_one_local_pass(qb):
    """A departing qubit at a low slot (< 2^4) is refilled by the highest
    staying qubit (physical_reorder_plan): one local transposition pass."""
    n, p = 10, 2
    lay = qb.QubitLayout.identity(n, qb.ClusterShape.flat(p))
    ev = qb.make_qr_event(lay, ((1 << n) - 1) & ~1)  # qubit 0 (slot 0) leaves, qubit 9 arrives
    dest, _ = qb.physical_reorder_plan(ev, list(range(n)))
    l0, l1, cross = qb.inplace_reorder_plan(n, p, dest)
    assert l0 == [(0, 8)] and not l1 and cross == [(8, 0)]


def test_three_cycle_takes_two_passes(qb):
    # rho = (0 -> 1 -> 2 -> 0) on local positions, no global move
    n, p = 6, 2
    dest = [1, 2, 0, 3, 4, 5]
    l0, l1, cross = qb.inplace_reorder_plan(n, p, dest)
    assert len(l0) == 1 and len(l1) == 1 and not cross
    sub = np.arange(2 * 32, dtype=np.complex128).reshape(2, 32)
    expect = np.empty_like(sub)
    for pe, (dpe, doff) in enumerate(push_map(qb, n, p, dest)):
        expect[dpe.astype(np.int64), doff.astype(np.int64)] = sub[pe]
    apply_local_pass(sub, l0, 5)
    apply_local_pass(sub, l1, 5)
    assert np.array_equal(sub, expect)


def test_global_to_global_rejected(qb):
    with pytest.raises(qb.Error):
        qb.inplace_reorder_plan(6, 4, [0, 1, 2, 3, 5, 4])
