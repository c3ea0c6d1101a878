"""BASELINE-config inputs pinned to the reference (CPU only).

tests/golden/configs.json is written by make_golden.py from the reference
itself (oracle/_ref):
* C4: HEA depth-20 schedules at 20/30/32/34 qubits, p = 2/4/8, lazy (flat) and
  eager (adhoc) — gate order, QR count and permutation sequence
  (qsu_scheduler.cpp:186-249) must match bit-exact;
* C5: the stress Hamiltonian, 10,000 words "IXYZ"[Rng(2024).below(4)]
  (models.cpp:26-35) with U(-1, 1) coefficients, and its EVC plans
  (evc_scheduler.cpp:238-280): 8,183 groups, 60 tiles, 59 QRs at 34q / p=8.
The GPU-side checks of the same configs live in tests/test_gpu_configs.py.
"""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

CFG = json.loads((GOLDEN / "configs.json").read_text())


def canon(obj):
    return json.dumps(obj, separators=(",", ":"), sort_keys=True)


def sha(obj):
    return hashlib.sha256(canon(obj).encode()).hexdigest()


@pytest.mark.parametrize("rec", CFG["hea_schedules"], ids=lambda r: f"{r['circuit']}-{r['shape']}-{r['scheduler']}")
def test_hea_schedule_matches_reference(qb, rec):
    _, n, depth = rec["circuit"].split(":")
    c = qb.gen_hea(int(n), int(depth), 1, False)
    d = qb.build_dependency_graph(c)
    fn = {"flat": qb.flat_tiling, "adhoc": qb.adhoc_schedule}[rec["scheduler"]]
    s = fn(c, d, qb.ClusterShape.flat(int(rec["shape"][4:])))
    counts = qb.count_qrs(s)
    assert counts.total == rec["counts"]["total"]
    assert len(s.tiles) == rec["tiles"]
    assert sha(json.loads(qb.schedule_to_json(s))) == rec["sha"]
    assert sha([list(ev.after.pos_of) for ev in s.qr_events]) == rec["events_sha"]


def test_hea_34_p8_counts():
    """34q HEA at p=8 — lazy 2 QRs, eager 259 (reference)."""
    by = {(r["circuit"], r["shape"], r["scheduler"]): r["counts"]["total"] for r in CFG["hea_schedules"]}
    assert by[("hea:34:20", "flat8", "flat")] == 2
    assert by[("hea:34:20", "flat8", "adhoc")] == 259


@pytest.mark.parametrize("rec", CFG["uniform_plans"], ids=lambda r: f"{r['terms']}-{r['shape']}")
def test_uniform_words_and_plan_match_reference(qb, rec):
    _, n, count, seed = rec["terms"].split(":")
    n, count, seed = int(n), int(count), int(seed)
    terms = qb.gen_uniform_words(n, count, seed)
    assert hashlib.sha256("".join(t.letters for t in terms).encode()).hexdigest() == rec["words_sha"]
    co = np.array([t.coeff for t in terms], dtype=np.complex128)
    assert hashlib.sha256(co.tobytes()).hexdigest() == rec["coeff_sha"]
    plan = qb.plan_evc(terms, n, qb.ClusterShape.flat(int(rec["shape"][4:])), rec["diag"], 8)
    assert len(qb.merge_terms(terms, rec["diag"])) == rec["groups"]
    assert len(plan.tiles) == rec["tiles"] and plan.qr_count() == rec["qr"]
    assert sha(json.loads(qb.plan_to_json(plan))) == rec["sha"]


def test_c5_survey_counts():
    """SURVEY.md §8d C5 stress: 8,183 groups, 60 tiles, 59 QRs at 34q / p=8."""
    rec = next(r for r in CFG["uniform_plans"] if r["terms"] == "uniform:34:10000:2024" and r["shape"] == "flat8")
    assert (rec["groups"], rec["tiles"], rec["qr"]) == (8183, 60, 59)


def test_c1_reference_totals():
    """C1 lazy 20 + 4 = 24 QRs, eager 159 + 5 = 164."""
    assert CFG["c1_flat"]["qsu_qr"] + CFG["c1_flat"]["evc_qr"] == 24
    assert CFG["c1_adhoc"]["qsu_qr"] + CFG["c1_adhoc"]["evc_qr"] == 164
    assert CFG["c1_flat"]["energy"] == -0.7999486529985721


def test_c1_product_qr_totals(qb):
    """The product's host layer reproduces C1's QR totals (QSU schedule + the EVC
    QRs re-derived from the post-QSU layout, dist_sim.cpp:268-271)."""
    n = 20
    c = qb.gen_gatefabric(n, 4 * n, 1, False)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(4)
    plan = qb.plan_evc(qb.gen_synthetic_jw(n, 1), n, shape, True, 8)
    for fn, key in ((qb.flat_tiling, "c1_flat"), (qb.adhoc_schedule, "c1_adhoc")):
        s = fn(c, d, shape)
        layout = s.qr_events[-1].after if len(s.qr_events) else qb.QubitLayout.identity(n, shape)
        evc = 0
        for tile in plan.tiles:
            ev = qb.make_qr_event(layout, tile.local_qubits)
            if ev is not None:
                evc += 1
                layout = ev.after
        assert qb.count_qrs(s).total == CFG[key]["qsu_qr"]
        assert evc == CFG[key]["evc_qr"]


def test_uniform_words_live_vs_reference(qb, ref):
    for n, count, seed in ((7, 50, 3), (34, 200, 2024), (12, 1, 9)):
        letters, co = ref.Terms.uniform(n, count, seed).export()
        mine = qb.gen_uniform_words(n, count, seed)
        assert letters == [t.letters for t in mine]
        assert np.array_equal(co, np.array([t.coeff for t in mine]))
