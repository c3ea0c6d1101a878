"""GPU parity at the BASELINE.json configs ("next round" item 1).

* C1 — the one config the reference's CPU path runs in full: 20-qubit
  GateFabric (layers 80, seed 1) + the full JW Hamiltonian (19,971 strings),
  flat(4), lazy (flat_tiling) and eager (adhoc_schedule).  The energy must be
  within 1e-10 * (1 + |E|) of the reference's evaluate_energy
  (dist_sim.cpp:357-363, tests/golden/configs.json) and the QSU + EVC QR totals
  must be the reference's 24 / 164.
* Cross-p invariance at 26 and 28 qubits (acceptance.cpp:287-309 at size):
  the same circuit on p = 1/2/4/8 PEs gives the same flattened state within
  1e-12 and the same energy within 1e-12 relative; lazy and eager agree too.
* C5's stress words (Rng(2024).below(4)) against the reference's expectation
  on small states, and cross-p invariance of their energy at 24 qubits.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CFG = json.loads((GOLDEN / "configs.json").read_text())
E_TOL = 1e-10


def run_iteration(qb, circuit, sched, terms, plan, n, shape):
    st = qb.init_state(n, shape)
    qb.run_qsu(st, circuit, sched)
    qsu = len(st.qr_log)
    e = qb.expectation(st, plan, terms)
    return st, e, qsu, len(st.qr_log) - qsu


@pytest.mark.parametrize("sched", ["flat", "adhoc"])
def test_c1_energy_and_qr_totals(qb, device, sched):
    n = 20
    c = qb.gen_gatefabric(n, 4 * n, 1, True)
    d = qb.build_dependency_graph(c)
    terms = qb.gen_synthetic_jw(n, 1)
    assert len(terms) == 19971
    shape = qb.ClusterShape.flat(4)
    s = (qb.flat_tiling if sched == "flat" else qb.adhoc_schedule)(c, d, shape)
    plan = qb.plan_evc(terms, n, shape, True, 8)
    gold = CFG[f"c1_{sched}"]
    st, e, qsu, evc = run_iteration(qb, c, s, terms, plan, n, shape)
    assert abs(e.real - gold["energy"]) <= E_TOL * (1 + abs(gold["energy"])), (e, gold["energy"])
    assert abs(e.imag) <= 1e-10
    assert (qsu, evc) == (gold["qsu_qr"], gold["evc_qr"])
    assert qsu + evc == (24 if sched == "flat" else 164)
    assert all(mv == qb.qr_data_volume(k, n) for k, mv in st.qr_log)
    # evaluate_energy (the public one-call iteration) gives the same number
    assert qb.evaluate_energy(c, s, terms, plan) == e.real


@pytest.mark.parametrize("n", [26, 28])
def test_cross_p_invariance(qb, device, n):
    """acceptance.cpp:287-309: state and energy independent of the PE count."""
    layers = 4 * n if n == 26 else 2 * n
    c = qb.gen_gatefabric(n, layers, 1, True)
    d = qb.build_dependency_graph(c)
    terms = qb.gen_synthetic_jw(n, 1, 10)
    ref_state, ref_e = None, None
    for p in (1, 2, 4, 8):
        shape = qb.ClusterShape.flat(p)
        plan = qb.plan_evc(terms, n, shape, True, 8)
        fns = (qb.flat_tiling, qb.adhoc_schedule) if (n == 26 and p in (1, 4)) else (qb.flat_tiling,)
        for fn in fns:
            s = fn(c, d, shape)
            st = qb.init_state(n, shape)
            qb.run_qsu(st, c, s)
            psi = qb.flatten(st)
            e = qb.expectation(st, plan, terms).real
            del st
            if ref_state is None:
                ref_state, ref_e = psi, e
                assert abs(np.linalg.norm(psi) - 1.0) <= 1e-12
                continue
            err = float(np.max(np.abs(psi - ref_state)))
            assert err <= 1e-12, (p, fn.__name__, err)
            assert abs(e - ref_e) <= 1e-12 * abs(ref_e), (p, fn.__name__, e, ref_e)
            del psi


@pytest.mark.parametrize("key", [k for k in CFG if k.startswith("evc_uniform_")])
def test_uniform_words_vs_reference(qb, device, key):
    _, _, n, count, rs, p = key.split("_")
    n, count, seed, p = int(n), int(count), int(rs[2:]), int(p[1:])
    terms = qb.gen_uniform_words(n, count, 2024)
    shape = qb.ClusterShape.flat(p)
    plan = qb.plan_evc(terms, n, shape, True, 4)
    st = qb.init_state_from(qb.random_state(n, seed), shape)
    got = qb.expectation(st, plan, terms)
    want = complex(*CFG[key]["energy"])
    assert abs(got - want) <= E_TOL * (1 + abs(want)), (got, want)
    assert len(st.qr_log) == CFG[key]["qr"]


def test_uniform_words_cross_p(qb, device):
    """C5 stress words at 24 qubits: the energy is independent of p (the
    plans differ: 1 tile at p=1, many QRs at p=8)."""
    n = 24
    terms = qb.gen_uniform_words(n, 2000, 2024)
    psi = qb.random_state(n, 1234)
    energies = []
    for p in (1, 2, 4, 8):
        shape = qb.ClusterShape.flat(p)
        plan = qb.plan_evc(terms, n, shape, True, 8)
        for _ in range(3 if p > 1 else 1):  # repeated: a pipeline race would show as run-to-run drift
            st = qb.init_state_from(psi, shape)
            energies.append(qb.expectation(st, plan, terms))
            if p > 1:
                assert len(st.qr_log) in (plan.qr_count(), plan.qr_count() + 1)
    for e in energies[1:]:
        assert abs(e - energies[0]) <= 1e-12 * (1 + abs(energies[0])), energies


@pytest.mark.parametrize("n,sched", [(24, "flat"), (24, "adhoc"), (26, "flat")])
def test_large_p8_energy_vs_reference(qb, device, n, sched):
    """Full 24- / 26-qubit iterations (GateFabric layers 4n, JW span-10, 8 PEs)
    against the reference's own evaluate_energy (tests/golden/configs.json,
    `make_golden.py large`): energy within 1e-10 * (1 + |E|) and the reference's
    QR counts."""
    key = f"c{n}_{sched}_p8"
    if key not in CFG:
        pytest.skip(f"{n}-qubit reference golden not generated")
    gold = CFG[key]
    c = qb.gen_gatefabric(n, 4 * n, 1, True)
    d = qb.build_dependency_graph(c)
    terms = qb.gen_synthetic_jw(n, 1, 10)
    shape = qb.ClusterShape.flat(8)
    s = (qb.flat_tiling if sched == "flat" else qb.adhoc_schedule)(c, d, shape)
    plan = qb.plan_evc(terms, n, shape, True, 8)
    st, e, qsu, evc = run_iteration(qb, c, s, terms, plan, n, shape)
    assert abs(e.real - gold["energy"]) <= E_TOL * (1 + abs(gold["energy"])), (e, gold["energy"])
    assert (qsu, evc) == (gold["qsu_qr"], gold["evc_qr"])
