"""N>1 host logic on CPU: 2, 4 or 8 gloo ranks (one per "GPU") emulate the
distributed QR exactly as libqrt performs it — PE ownership (rank r owns PEs
[r*p/w, (r+1)*p/w)), the physical placement chosen by physical_reorder_plan,
and the kernel's own destination mapping replayed by qrt_reorder_plan — and
exchange amplitudes with torch.distributed.  Results must equal the oracle's
perform_qr (dist_sim.cpp:203-240) bit for bit, and relocation counts must
equal qr_data_volume.
"""
import ctypes as C
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan(lib, n, p, dest, pe):
    per = 1 << (n - (p.bit_length() - 1))
    dpe = np.zeros(per, dtype=np.uint64)
    doff = np.zeros(per, dtype=np.uint64)
    rel = C.c_uint64()
    rc = lib.qrt_reorder_plan(n, p, (C.c_int * n)(*dest), pe, dpe.ctypes.data_as(C.POINTER(C.c_uint64)),
                              doff.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(rel))
    assert rc == 0
    return dpe, doff, rel.value


def _exchange_inplace(dist, rank, world, per_rank, mine, local, nl, p, cross):
    """exchange_kernel over gloo: PE j's class s swaps with PE s's class j; the
    pair's lower PE handles the half with bit f = 0 (qrt_reorder.cu).  Remote
    reads come from an all-gather of the old buffers, remote writes travel to
    the owning rank; every amplitude must be written exactly once."""
    k = len(cross)
    d = [c[0] for c in cross]
    pb = [c[1] for c in cross]
    f = max((x for x in range(nl) if x not in set(d)), default=-1)
    gathered = [None] * world
    dist.all_gather_object(gathered, {pe: local[pe] for pe in mine})
    old = {pe: buf for g in gathered for pe, buf in g.items()}
    o = np.arange(1 << nl, dtype=np.uint64)
    cls = np.zeros(o.shape, dtype=np.int64)
    for i in range(k):
        cls |= ((o >> np.uint64(d[i])) & np.uint64(1)).astype(np.int64) << i
    new = {pe: local[pe].copy() for pe in mine}
    touched = {pe: np.zeros(1 << nl, dtype=np.int64) for pe in mine}
    remote = [[] for _ in range(world)]
    for j in mine:
        jc = sum(((j >> pb[i]) & 1) << i for i in range(k))
        for s in range(1 << k):
            if s == jc:
                continue
            sp = j
            for i in range(k):
                sp = (sp & ~(1 << pb[i])) | (((s >> i) & 1) << pb[i])
            sel = cls == s
            if f >= 0:
                sel &= ((o >> np.uint64(f)) & np.uint64(1)) == np.uint64(0 if j < sp else 1)
            elif j > sp:
                continue
            a = o[sel]
            b = a.copy()
            for i in range(k):
                b = (b & ~(np.uint64(1) << np.uint64(d[i]))) | (np.uint64((jc >> i) & 1) << np.uint64(d[i]))
            new[j][a.astype(np.int64)] = old[sp][b.astype(np.int64)]  # remote read, local store
            touched[j][a.astype(np.int64)] += 1
            remote[sp // per_rank].append((sp, b, old[j][a.astype(np.int64)]))  # remote store
    for r in range(world):
        box = [None] * world
        dist.all_gather_object(box, remote[r])
        if r == rank:
            for sent in box:
                for sp, b, vals in sent:
                    new[sp][b.astype(np.int64)] = vals
                    touched[sp][b.astype(np.int64)] += 1
    ok = all(int(t.max()) <= 1 for t in touched.values())
    return new, ok


def _worker(rank, world, port, n, p, seed, q, mode="push"):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2410_04252_b200 as qb
    from oracle import cpu

    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = qb.load_libqrt()
    per_rank = p // world
    mine = list(range(rank * per_rank, (rank + 1) * per_rank))
    psi = qb.random_state(n, seed)
    sub_all = psi.reshape(p, -1).copy()           # oracle copy (every rank)
    local = {pe: sub_all[pe].copy() for pe in mine}  # this rank's PEs, physical order
    layout = qb.QubitLayout.identity(n, qb.ClusterShape.flat(p))
    phys = list(range(n))
    olay = cpu.Layout(n, p)
    rng = np.random.default_rng(seed)
    ok = True
    for _ in range(4):
        locals_ = 0
        while bin(locals_).count("1") < layout.n_local:
            locals_ |= 1 << int(rng.integers(n))
        ev = qb.make_qr_event(layout, locals_)
        if ev is None:
            continue
        dest, new_phys = qb.physical_reorder_plan(ev, phys)
        if mode == "inplace":
            # the in-place QR: local transposition passes on every PE, then the
            # pairwise slot-class exchange (qrt_reorder_inplace_plan)
            from test_inplace_qr import apply_local_pass
            l0, l1, cross = qb.inplace_reorder_plan(n, p, dest)
            nl0 = n - (p.bit_length() - 1)
            for pe in mine:
                buf = local[pe].reshape(1, -1).copy()
                apply_local_pass(buf, l0, nl0)
                apply_local_pass(buf, l1, nl0)
                local[pe] = buf[0]
            local, once = _exchange_inplace(dist, rank, world, per_rank, mine, local, nl0, p, cross)
            ok = ok and once
            _, _, rel_seen = _plan(lib, n, p, dest, mine[0])
        else:
            # emulate the push kernel: each local PE sends every amplitude to (dst_pe, dst_off)
            outgoing = [[] for _ in range(world)]
            rel_seen = None
            for pe in mine:
                dpe, doff, rel = _plan(lib, n, p, dest, pe)
                rel_seen = rel
                for r in range(world):
                    sel = (dpe // per_rank) == r
                    outgoing[r].append((dpe[sel], doff[sel], local[pe][sel]))
            incoming = [None] * world
            for r in range(world):
                gathered = [None] * world
                dist.all_gather_object(gathered, outgoing[r])
                incoming[r] = gathered  # what every rank sends to rank r
            fresh = {pe: np.zeros_like(local[pe]) for pe in mine}
            for src_rank in range(world):
                for dpe, doff, vals in incoming[rank][src_rank]:
                    for pe in mine:
                        sel = dpe == pe
                        fresh[pe][doff[sel].astype(np.int64)] = vals[sel]
            local = fresh
        moved = cpu.perform_qr(sub_all, olay.dest_for(ev.after.pos_of))
        olay.adopt(ev.after.pos_of)
        ok = ok and rel_seen == moved == qb.qr_data_volume(len(ev.swaps), n)
        # compare in reference (logical) position order
        nl = layout.n_local
        layout = ev.after
        phys = new_phys
        lp = [phys[layout.qubit_at[pos]] for pos in range(nl)]
        idx = np.zeros(1 << nl, dtype=np.int64)
        for pos, ph in enumerate(lp):
            idx |= ((np.arange(1 << nl) >> pos) & 1) << ph
        for pe in mine:
            ok = ok and np.array_equal(local[pe][idx], sub_all[pe])
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["push", "inplace"])
@pytest.mark.parametrize("world,n,p,seed", [(2, 8, 2, 1), (2, 10, 4, 2), (2, 11, 8, 3), (4, 10, 4, 4), (8, 12, 8, 5)])
def test_multi_rank_reorder_matches_oracle(world, n, p, seed, mode):
    """world = 8, p = 8 is the one-PE-per-GPU layout of an 8xB200 box (every
    lazy QR there swaps all three global bits: an 8-way all-to-all).  `inplace`
    replays the single-buffer QR: local transposition passes + the pairwise
    class exchange with its f-bit ownership split across ranks."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, p, seed, q, mode)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert results == {r: True for r in range(world)}
