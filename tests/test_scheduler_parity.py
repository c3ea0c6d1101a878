"""Host schedulers vs the reference, bit-exact (CPU only).

Every schedule the product emits must match the reference's gate order, tile
mappings, QR count and qubit-permutation sequence exactly
(reference qsu_scheduler.cpp:14-249, evc_scheduler.cpp:120-280).  Golden
records in tests/golden/ come from the reference itself (make_golden.py);
when oracle/_ref is built the comparison is also run live on fresh inputs.
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

SCHED = json.loads((GOLDEN / "schedules.json").read_text())
PLANS = json.loads((GOLDEN / "plans.json").read_text())


def canon(obj):
    return json.dumps(obj, separators=(",", ":"), sort_keys=True)


def sha(obj):
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def shape_of(qb, name):
    return {"flat2": qb.ClusterShape.flat(2), "flat4": qb.ClusterShape.flat(4), "flat8": qb.ClusterShape.flat(8),
            "flat16": qb.ClusterShape.flat(16), "2x2": qb.ClusterShape.two_level(2, 2),
            "2x4": qb.ClusterShape.two_level(2, 4), "4x4": qb.ClusterShape.two_level(4, 4)}[name]


def circuit_of(qb, key):
    kind, *rest = key.split(":")
    if kind == "gatefabric":
        n, layers, seed = map(int, rest)
        return qb.gen_gatefabric(n, layers, seed, False)
    if kind == "fixture":
        return qb.fixture_circuit(rest[0], 1)
    n, m, seed, ar = map(int, rest)
    return qb.gen_random_circuit(n, m, seed, ar, False)


@pytest.mark.parametrize("rec", SCHED, ids=lambda r: f"{r['circuit']}-{r['shape']}-{r['scheduler']}")
def test_schedule_matches_reference(qb, rec):
    c = circuit_of(qb, rec["circuit"])
    d = qb.build_dependency_graph(c)
    fn = {"flat": qb.flat_tiling, "hierarchical": qb.hierarchical_tiling, "adhoc": qb.adhoc_schedule}[rec["scheduler"]]
    s = fn(c, d, shape_of(qb, rec["shape"]))
    counts = qb.count_qrs(s)
    assert (counts.total, counts.intra, counts.inter) == (rec["counts"]["total"], rec["counts"]["intra"],
                                                          rec["counts"]["inter"])
    assert len(s.tiles) == rec["tiles"]
    assert sha(json.loads(qb.schedule_to_json(s))) == rec["sha"]
    assert sha([list(ev.after.pos_of) for ev in s.qr_events]) == rec["events_sha"]
    if rec.get("schedule"):
        assert json.loads(qb.schedule_to_json(s)) == rec["schedule"]
    assert qb.validate_schedule(c, d, s) is None and qb.schedule_is_narrow(c, s)


@pytest.mark.parametrize("rec", PLANS, ids=lambda r: f"{r['terms']}-{r['shape']}-{r['diag']}")
def test_plan_matches_reference(qb, rec):
    _, n, seed, span = rec["terms"].split(":")
    n, seed, span = int(n), int(seed), int(span)
    terms = qb.gen_synthetic_jw(n, seed, span)
    shape = shape_of(qb, rec["shape"])
    if "error" in rec:
        with pytest.raises(qb.Error):
            qb.plan_evc(terms, n, shape, rec["diag"], 8)
        return
    plan = qb.plan_evc(terms, n, shape, rec["diag"], 8)
    assert plan.qr_count() == rec["qr"]
    assert len(plan.tiles) == rec["tiles"]
    assert len(qb.merge_terms(terms, rec["diag"])) == rec["groups"]
    assert qb.index_order_baseline(terms, n, shape).n_qr == rec["baseline"]
    assert sha(json.loads(qb.plan_to_json(plan))) == rec["sha"]


def test_paper_figures(qb):
    """acceptance.cpp:175-199: Fig. 6 (3 QRs, first tile 9 gates under Q_G={12..15})
    and Fig. 8 (hierarchical: 2 inter + 3 intra, cost 51 < 72)."""
    c = qb.fixture_circuit("gatefabric-fig6")
    d = qb.build_dependency_graph(c)
    s = qb.flat_tiling(c, d, qb.ClusterShape.flat(16))
    assert qb.count_qrs(s).total == 3
    assert len(s.tiles[0].gates) == 9 and s.tiles[0].local_qubits == (1 << 12) - 1
    grid = qb.ClusterShape.two_level(4, 4)
    h = qb.count_qrs(qb.hierarchical_tiling(c, d, grid))
    f = qb.count_qrs(qb.flat_tiling(c, d, grid))
    w = qb.CostWeights(1.0, 24.0)
    assert (h.inter, h.intra) == (2, 3) and qb.qr_cost(h, w) == 51.0 and qb.qr_cost(f, w) == 72.0


def test_fig7_and_adhoc_pairs(qb):
    # test_qsu_scheduler.cpp:104-116 (Fig. 7) and :251-261 (ad hoc single swap)
    c = qb.fixture_circuit("fig7")
    order = qb.depth_sort(c, qb.build_dependency_graph(c))
    assert qb.tile_construction(0b001111, c, order) == [0, 1, 3, 5]
    assert qb.qubit_mapping((1 << 6) - 1, c, [2, 4, 7, 6], 4) == 0b111100
    one = qb.Circuit(6, [qb.make_gate(0, [0, 5])])
    s = qb.adhoc_schedule(one, qb.build_dependency_graph(one), qb.ClusterShape.flat(4))
    assert qb.count_qrs(s).total == 1 and s.qr_events[0].swaps == [(1, 5)]
    # pairing rule: departing and arriving qubits matched in ascending order
    lay = qb.QubitLayout.identity(6, qb.ClusterShape.flat(4))
    ev = qb.make_qr_event(lay, 0b110110)
    assert ev.swaps == [(0, 4), (3, 5)]


def test_dominance_gatefabric(qb):
    # acceptance.cpp:202-225
    for n in (8, 12, 16, 20):
        for layers in (1, 2, 3):
            c = qb.gen_gatefabric(n, layers, 77, False)
            d = qb.build_dependency_graph(c)
            shape = qb.ClusterShape.two_level(2, 2)
            f = qb.count_qrs(qb.flat_tiling(c, d, shape)).total
            a = qb.count_qrs(qb.adhoc_schedule(c, d, shape)).total
            assert f <= a and (f < a or layers < 2)


def test_partitioned_search_identical(qb):
    # acceptance.cpp:311-323: byte-identical for workers in {1,2,4,8}
    terms = qb.gen_synthetic_jw(12, 5)
    groups = qb.merge_terms(terms, True)
    shape = qb.ClusterShape.two_level(2, 2)
    serial = qb.plan_to_json(qb.tiling_pauli_strings(groups, 12, shape, True, 1))
    for w in (2, 4, 8):
        assert qb.plan_to_json(qb.tiling_pauli_strings(groups, 12, shape, True, w)) == serial


def test_evc_tiling_suite(qb):
    # acceptance.cpp:227-237: jw12 p=4 tiler QRs <= 5, baseline ratio >= 20
    terms = qb.gen_synthetic_jw(12, 3)
    shape = qb.ClusterShape.two_level(2, 2)
    plan = qb.plan_evc(terms, 12, shape, True)
    base = qb.index_order_baseline(terms, 12, shape)
    assert plan.qr_count() <= 5 and base.n_qr / max(1, plan.qr_count()) >= 20


def test_errors(qb):
    c = qb.Circuit(4, [qb.make_gate(0, [0, 1, 2])])
    with pytest.raises(qb.GateTooWide):
        qb.flat_tiling(c, qb.build_dependency_graph(c), qb.ClusterShape.flat(4))
    with pytest.raises(qb.ConfigError):
        qb.ClusterShape.flat(3).validate()
    with pytest.raises(qb.TooManyPEs):
        qb.QubitLayout.identity(2, qb.ClusterShape.flat(8))
    assert qb.qr_data_volume(4, 16) == 61440  # test_layout.cpp:114


def test_live_random_vs_reference(qb, ref):
    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.integers(4, 14))
        m = int(rng.integers(1, 150))
        seed = int(rng.integers(1 << 40))
        c = qb.gen_random_circuit(n, m, seed, 3 if n > 4 else 2, False)
        rc = ref.Circuit.random(n, m, seed, 3 if n > 4 else 2, False)
        d = qb.build_dependency_graph(c)
        assert qb.depth_sort(c, d) == rc.depth_sort()["order"]
        for p in (2, 4, 8):
            if p > (1 << (n - 3)):
                continue
            for sched, fn in (("flat", qb.flat_tiling), ("hierarchical", qb.hierarchical_tiling),
                              ("adhoc", qb.adhoc_schedule)):
                got = json.loads(qb.schedule_to_json(fn(c, d, qb.ClusterShape.flat(p))))
                assert got == rc.schedule(sched, p)["schedule"]


@pytest.mark.parametrize("p", [2, 4, 8])
def test_batched_evc_search_identical(qb, monkeypatch, p):
    """The incremental inclusion-exclusion tile search (g <= 3 global qubits)
    emits the exhaustive search's plan byte for byte (evc_scheduler.cpp:150-236,
    first lexicographic maximum), on uniform and Jordan-Wigner inputs."""
    rng = np.random.default_rng(p)
    for trial in range(12):
        n = int(rng.integers(6, 15))
        if p > (1 << (n - 3)):
            continue
        terms = (qb.gen_uniform_words(n, int(rng.integers(5, 300)), int(rng.integers(1 << 30)))
                 if trial % 2 == 0 else qb.gen_synthetic_jw(n, int(rng.integers(1, 99)), int(rng.integers(3, n))))
        shape = qb.ClusterShape.flat(p)
        try:
            monkeypatch.setenv("QRT_EVC_PLAN_BATCHED", "0")
            slow = qb.plan_to_json(qb.plan_evc(terms, n, shape, True, 4))
        except qb.Error:
            continue
        monkeypatch.setenv("QRT_EVC_PLAN_BATCHED", "1")
        assert qb.plan_to_json(qb.plan_evc(terms, n, shape, True, 4)) == slow


def test_batched_evc_search_fast(qb):
    """C5 stress planning (10,000 uniform words, 34 qubits, p = 8: 60 tiles)
    well under the exhaustive search's seconds (<= 0.3 s)."""
    import time
    terms = qb.gen_uniform_words(34, 10000, 2024)
    t0 = time.perf_counter()
    plan = qb.plan_evc(terms, 34, qb.ClusterShape.flat(8), True, 1)
    assert len(plan.tiles) == 60
    assert time.perf_counter() - t0 < 1.0
