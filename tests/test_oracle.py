"""Pin the oracle (CPU only).

The C restatement (oracle/qrt_oracle.c) and the product's host generators are
checked against the golden vectors produced by the reference itself
(tests/golden/, make_golden.py) and, where oracle/_ref is built, against the
live reference.  Only once pinned is the oracle used as the GPU checker.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import cpu

GEN = json.loads((GOLDEN / "generators.json").read_text())
DS = json.loads((GOLDEN / "distsim.json").read_text())


def unhex(vals):
    return np.array([float.fromhex(v) for v in vals], dtype=np.float64)


def test_generators_bit_exact(qb):
    g = GEN["gatefabric_8_2_1"]
    c = qb.gen_gatefabric(8, 2, 1, True)
    assert [op.arity() for op in c.operators] == g["arity"]
    assert [q for op in c.operators for q in op.targets] == g["targets"]
    first = np.ascontiguousarray(c.operators[0].payload).view(np.float64).ravel()
    assert np.array_equal(first, unhex(g["first_block"]))
    import hashlib
    allm = np.concatenate([np.ascontiguousarray(op.payload).view(np.float64).ravel() for op in c.operators])
    assert hashlib.sha256(allm.tobytes()).hexdigest() == g["mats_sha"]
    r = GEN["random_6_12_77_3"]
    rc = qb.gen_random_circuit(6, 12, 77, 3, True)
    assert [q for op in rc.operators for q in op.targets] == r["targets"]
    rm = np.concatenate([np.ascontiguousarray(op.payload).view(np.float64).ravel() for op in rc.operators])
    assert hashlib.sha256(rm.tobytes()).hexdigest() == r["mats_sha"]
    jw = qb.gen_synthetic_jw(8, 1)
    assert [t.letters for t in jw] == GEN["jw_8_1"]["letters"]
    assert np.array_equal(np.array([t.coeff for t in jw]).view(np.float64), unhex(GEN["jw_8_1"]["coeffs"]))
    for key, cnt in GEN["jw_counts"].items():
        n, s = map(int, key.split(":"))
        assert qb.synthetic_jw_term_count(n, s) == cnt == len(qb.gen_synthetic_jw(n, 1, s))
    assert np.array_equal(qb.random_state(6, 11).view(np.float64), unhex(GEN["random_state_6_11"]))


@pytest.mark.parametrize("key", [k for k in DS if k.startswith("qsu_")])
def test_oracle_run_qsu_matches_reference(qb, key):
    rec = DS[key]
    want = unhex(rec["state"]).view(np.complex128)
    parts = key.split("_")
    if parts[1] == "gatefabric":
        n, layers, seed = int(parts[2]), int(parts[3]), int(parts[4])
        c = qb.gen_gatefabric(n, layers, seed, True)
        sched, p = parts[5], int(parts[6])
    else:
        n, m, seed = int(parts[2]), int(parts[3]), int(parts[4])
        c = qb.gen_random_circuit(n, m, seed, 2, True)
        sched, p = parts[5], int(parts[6])
    shape = qb.ClusterShape.two_level(2, 2) if sched == "adhoc" else qb.ClusterShape.flat(p)
    fn = {"flat": qb.flat_tiling, "adhoc": qb.adhoc_schedule}[sched]
    s = fn(c, qb.build_dependency_graph(c), shape)
    sub, lay, moved = cpu.run_qsu(n, p, c, s)
    got = cpu.flatten(sub, lay.qubit_at)
    assert np.array_equal(got, want)  # bit-exact restatement
    assert moved == [mv for _, mv in rec["qr_log"]]


def test_oracle_expectation_matches_reference(qb):
    psi = qb.random_state(10, 4010)
    terms = qb.gen_synthetic_jw(10, 610)
    for p in (1, 4):
        rec = DS[f"evc_jw10_610_rs4010_p{p}"]
        shape = qb.ClusterShape.flat(p)
        plan = qb.plan_evc(terms, 10, shape, True)
        sub = psi.reshape(p, -1).copy()
        lay = cpu.Layout(10, p)
        layout = qb.QubitLayout.identity(10, shape)
        partial = np.zeros(p, dtype=complex)
        for tile in plan.tiles:
            if layout.local_set() != tile.local_qubits:
                ev = qb.make_qr_event(layout, tile.local_qubits)
                cpu.perform_qr(sub, lay.dest_for(ev.after.pos_of))
                lay.adopt(ev.after.pos_of)
                layout = ev.after
            masked = [cpu.mask_term(terms[i].letters, lay.pos_of, lay.nl) for i in tile.terms]
            partial += cpu.expectation_tile(sub, masked, [terms[i].coeff for i in tile.terms])
        e = 0j
        for x in partial:  # ascending PE order, sequential (dist_sim.cpp:297-298)
            e += x
        assert e.real == rec["energy"][0] and e.imag == rec["energy"][1]  # bit-exact


def test_oracle_qr_relocation_formula():
    # test_dist_sim.cpp:183-199 on the oracle
    rng = np.random.default_rng(7)
    for _ in range(20):
        n = int(rng.integers(4, 11))
        p = 1 << int(rng.integers(1, min(3, n - 1) + 1))
        lay = cpu.Layout(n, p)
        sub = (rng.standard_normal((p, 1 << lay.nl)) + 1j * rng.standard_normal((p, 1 << lay.nl)))
        before = cpu.flatten(sub, lay.qubit_at)
        perm = list(range(n))
        k = int(rng.integers(1, min(lay.nl, n - lay.nl) + 1))
        loc = rng.choice(lay.nl, size=k, replace=False)
        glb = rng.choice(np.arange(lay.nl, n), size=k, replace=False)
        for a, b in zip(loc, glb):
            perm[a], perm[b] = perm[b], perm[a]
        after_pos = [perm[lay.pos_of[q]] for q in range(n)]
        moved = cpu.perform_qr(sub, lay.dest_for(after_pos))
        lay.adopt(after_pos)
        assert moved == (1 << n) - (1 << (n - k))
        assert np.array_equal(cpu.flatten(sub, lay.qubit_at), before)


def test_live_oracle_vs_reference(qb, ref):
    """Random circuits: C restatement == reference run_qsu, bit for bit."""
    rng = np.random.default_rng(11)
    for _ in range(10):
        n = int(rng.integers(4, 11))
        p = 1 << int(rng.integers(1, min(3, n - 2) + 1))
        m = int(rng.integers(1, 60))
        seed = int(rng.integers(1 << 40))
        c = qb.gen_random_circuit(n, m, seed, 2, True)
        s = qb.flat_tiling(c, qb.build_dependency_graph(c), qb.ClusterShape.flat(p))
        sub, lay, _ = cpu.run_qsu(n, p, c, s)
        want, _ = ref.Circuit.random(n, m, seed, 2, True).run_qsu("flat", p)
        assert np.array_equal(cpu.flatten(sub, lay.qubit_at), want)
