"""In-place QR on the GPU (QRT_QR_INPLACE=1): one buffer per PE, local
bit-transposition passes + the pairwise slot-class swap (csrc/qrt_reorder.cu
execute_inplace).  A QR is a pure permutation, so the
in-place path must give bit-identical states to the push exchange and match
the oracle's perform_qr (dist_sim.cpp:203-240) exactly.
"""
import numpy as np
import pytest

from oracle import cpu

pytestmark = pytest.mark.gpu


@pytest.fixture
def inplace(monkeypatch):
    monkeypatch.setenv("QRT_QR_INPLACE", "1")


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("sched", ["flat", "adhoc"])
def test_qsu_inplace_matches_oracle(qb, device, inplace, p, sched):
    n = 14
    c = qb.gen_gatefabric(n, 3 * n, 5, True)
    d = qb.build_dependency_graph(c)
    s = (qb.flat_tiling if sched == "flat" else qb.adhoc_schedule)(c, d, qb.ClusterShape.flat(p))
    st = qb.init_state(n, qb.ClusterShape.flat(p))
    assert qb.state_mode(st)["inplace_qr"]
    qb.run_qsu(st, c, s)
    sub, lay, moved = cpu.run_qsu(n, p, c, s)
    want = cpu.flatten(sub, lay.qubit_at)
    got = qb.flatten(st)
    assert float(np.max(np.abs(got - want))) <= 1e-12
    assert [m for _, m in st.qr_log] == moved


def test_hea_inplace_matches_oracle(qb, device, inplace):
    n, p = 13, 8
    c = qb.gen_hea(n, 6, 2, True)
    d = qb.build_dependency_graph(c)
    s = qb.adhoc_schedule(c, d, qb.ClusterShape.flat(p))
    st = qb.init_state(n, qb.ClusterShape.flat(p))
    qb.run_qsu(st, c, s)
    sub, lay, _ = cpu.run_qsu(n, p, c, s)
    assert float(np.max(np.abs(qb.flatten(st) - cpu.flatten(sub, lay.qubit_at)))) <= 1e-12


@pytest.mark.parametrize("p", [2, 4])
def test_inplace_bit_identical_to_push(qb, device, monkeypatch, p):
    """Same circuit, same schedule: a single-buffer state (every QR in place)
    and a two-buffer state (QRs fused into the next gate pass where possible)
    give identical bits (the QR is a permutation; the gate passes see the
    same physical layout)."""
    n = 22
    c = qb.gen_gatefabric(n, 2 * n, 1, True)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(p)
    s = qb.adhoc_schedule(c, d, shape)
    terms = qb.gen_synthetic_jw(n, 1, 10)
    plan = qb.plan_evc(terms, n, shape, True, 8)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("QRT_QR_INPLACE", mode)
        st = qb.init_state(n, shape)
        assert qb.state_mode(st)["inplace_qr"] == (mode == "1")
        qb.run_qsu(st, c, s)
        psi = qb.flatten(st)
        e = qb.expectation(st, plan, terms)
        out[mode] = (psi, e, list(st.qr_log))
        del st
    assert np.array_equal(out["0"][0], out["1"][0])
    assert out["0"][1] == out["1"][1]
    assert out["0"][2] == out["1"][2]


def test_inplace_large_roundtrip(qb, device, inplace):
    """26 qubits on 4 PEs: k = 2 QR there and back is bit-exact in place; a QR
    departing slot 0 (refill: one local pass) too."""
    n, p = 26, 4
    st = qb.init_state(n, qb.ClusterShape.flat(p))
    c = qb.gen_gatefabric(n, 2, 3, True)
    ids = [op.id for op in c.operators if all(q < n - 2 for q in op.targets)]
    qb.apply_gates_narrow(st, c, ids)
    before = [st.sub_of(pe) for pe in range(p)]
    locals0 = st.layout.local_set()
    for gone in (0b11 << 10, 0b11):  # slots 10/11 (pure swap), then slots 0/1 (refilled)
        ev = qb.make_qr_event(st.layout, (((1 << (n - 2)) - 1) & ~gone) | (0b11 << (n - 2)))
        qb.perform_qr(st, ev)
        assert st.last_relocated == qb.qr_data_volume(2, n)
        back = qb.make_qr_event(st.layout, locals0)
        qb.perform_qr(st, back)
        for pe in range(p):
            assert np.array_equal(st.sub_of(pe), before[pe])
    assert abs(st.norm() - 1.0) <= 1e-12


def test_c1_inplace(qb, device, inplace):
    """C1 (20q GateFabric, full JW, flat(4)) through the in-place QR path:
    the reference's energy and 24 QRs."""
    import json

    from conftest import GOLDEN
    gold = json.loads((GOLDEN / "configs.json").read_text())["c1_flat"]
    n = 20
    c = qb.gen_gatefabric(n, 4 * n, 1, True)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(4)
    terms = qb.gen_synthetic_jw(n, 1)
    s = qb.flat_tiling(c, d, shape)
    plan = qb.plan_evc(terms, n, shape, True, 8)
    st = qb.init_state(n, shape)
    qb.run_qsu(st, c, s)
    e = qb.expectation(st, plan, terms).real
    assert abs(e - gold["energy"]) <= 1e-10 * (1 + abs(gold["energy"]))
    assert len(st.qr_log) == 24
