"""Regenerate tests/golden/*.json from the *reference itself*.

Runs the unmodified reference library (oracle/_ref/libqrtile_ref.so, built by
oracle/Makefile from /root/reference sources) and records the values the
product must reproduce:

* schedules  (qsu_scheduler.cpp): counts and sha256 of schedule_to_json for
  GateFabric at the BASELINE configs (20/30/32/34 qubits, p = 2/4/8, flat /
  hierarchical / adhoc, flat(p) and two_level shapes) and the paper fixtures;
* EVC plans  (evc_scheduler.cpp): sha256 of plan_to_json, QR and baseline counts;
* generators (models.cpp): exact payload / coefficient / state bits;
* dist-sim   (dist_sim.cpp): small QSU output states, expectations, energies;
* configs    the BASELINE configs: C1 energies and QR totals (20q, 4 PEs, lazy
  and eager), C4 HEA schedules, C5 uniform-word plans (Rng(2024)).

    python tests/golden/make_golden.py        # needs oracle/_ref (make -C oracle ref)
    python tests/golden/make_golden.py configs   # only configs.json
    python tests/golden/make_golden.py large     # + the 24-qubit reference iterations
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import ref as R  # noqa: E402


def canon(obj) -> str:
    return json.dumps(obj, separators=(",", ":"), sort_keys=True)


def sha(obj) -> str:
    return hashlib.sha256(canon(obj).encode()).hexdigest()


def shapes():
    yield "flat2", (2, 0, 0)
    yield "flat4", (4, 0, 0)
    yield "flat8", (8, 0, 0)
    yield "2x2", (0, 2, 2)
    yield "2x4", (0, 2, 4)


def schedules():
    out = []
    for n in (8, 12, 16, 20, 30, 32, 34):
        c = R.Circuit.gatefabric(n, 4 * n, 1, False)
        for sname, (p, nn, ng) in shapes():
            if p == 0:
                p = nn * ng
            for sched in ("flat", "hierarchical", "adhoc"):
                d = c.schedule(sched, p, nn, ng)
                out.append({"circuit": f"gatefabric:{n}:{4 * n}:1", "shape": sname, "scheduler": sched,
                            "counts": d["counts"], "tiles": len(d["schedule"]["tiles"]),
                            "sha": sha(d["schedule"]),
                            "events_sha": sha([e["after_pos_of"] for e in d["events"]])})
    for name in ("fig2", "fig3", "fig7", "gatefabric-fig6"):
        c = R.Circuit.fixture(name, 1)
        for sname, (p, nn, ng) in [("flat4", (4, 0, 0)), ("flat16", (16, 0, 0)), ("4x4", (0, 4, 4))]:
            if p == 0:
                p = nn * ng
            if name != "gatefabric-fig6" and p > 4:
                continue
            for sched in ("flat", "hierarchical", "adhoc"):
                d = c.schedule(sched, p, nn, ng)
                out.append({"circuit": f"fixture:{name}", "shape": sname, "scheduler": sched,
                            "counts": d["counts"], "tiles": len(d["schedule"]["tiles"]),
                            "schedule": d["schedule"] if name != "gatefabric-fig6" else None,
                            "sha": sha(d["schedule"]),
                            "events_sha": sha([e["after_pos_of"] for e in d["events"]])})
    for seed in range(20):
        c = R.Circuit.random(4 + seed % 9, 1 + (7 * seed) % 99, 1000 + seed, 2, False)
        for sname, (p, nn, ng) in [("flat2", (2, 0, 0)), ("2x2", (0, 2, 2))]:
            if p == 0:
                p = nn * ng
            for sched in ("flat", "hierarchical", "adhoc"):
                d = c.schedule(sched, p, nn, ng)
                out.append({"circuit": f"random:{4 + seed % 9}:{1 + (7 * seed) % 99}:{1000 + seed}:2",
                            "shape": sname, "scheduler": sched, "counts": d["counts"],
                            "tiles": len(d["schedule"]["tiles"]), "sha": sha(d["schedule"]),
                            "events_sha": sha([e["after_pos_of"] for e in d["events"]])})
    return out


def plans():
    out = []
    for n, span in ((8, 0), (12, 0), (12, 10), (20, 10), (30, 10), (34, 10)):
        t = R.Terms.jw(n, 1, span)
        for sname, (p, nn, ng) in shapes():
            if p == 0:
                p = nn * ng
            for diag in (True, False):
                if not diag and span == 0 and n > 8:
                    continue
                try:
                    d = t.plan(n, p, nn, ng, diag, 8)
                except RuntimeError as e:
                    out.append({"terms": f"jw:{n}:1:{span}", "shape": sname, "diag": diag, "error": str(e)[:60]})
                    continue
                out.append({"terms": f"jw:{n}:1:{span}", "shape": sname, "diag": diag, "qr": d["qr_count"],
                            "baseline": d["baseline_qr"], "groups": d["n_groups"], "tiles": len(d["plan"]["tiles"]),
                            "sha": sha(d["plan"])})
    return out


def hexs(a: np.ndarray):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def generators():
    c = R.Circuit.gatefabric(8, 2, 1, True)
    ar, tg, mats = c.export()
    rc = R.Circuit.random(6, 12, 77, 3, True)
    rar, rtg, rmats = rc.export()
    letters, co = R.Terms.jw(8, 1, 0).export()
    return {
        "gatefabric_8_2_1": {"arity": ar.tolist(), "targets": tg.tolist(), "mats_sha": hashlib.sha256(mats.tobytes()).hexdigest(),
                             "first_block": hexs(mats[:512])},
        "random_6_12_77_3": {"arity": rar.tolist(), "targets": rtg.tolist(),
                             "mats_sha": hashlib.sha256(rmats.tobytes()).hexdigest()},
        "jw_8_1": {"letters": letters, "coeffs": hexs(co.view(np.float64))},
        "jw_counts": {f"{n}:{s}": len(R.Terms.jw(n, 1, s).export()[0]) for n, s in ((20, 0), (30, 10), (32, 10), (34, 10))},
        "random_state_6_11": hexs(R.random_state(6, 11).view(np.float64)),
    }


def distsim():
    out = {}
    c = R.Circuit.gatefabric(8, 3, 5, True)
    for sched, (p, nn, ng) in (("flat", (4, 0, 0)), ("adhoc", (0, 2, 2))):
        if p == 0:
            p = nn * ng
        st, log = c.run_qsu(sched, p, nn, ng, 1)
        out[f"qsu_gatefabric_8_3_5_{sched}_{p}"] = {"state": hexs(st.view(np.float64)), "qr_log": log}
    rc = R.Circuit.random(7, 40, 99, 2, True)
    st, log = rc.run_qsu("flat", 4, 0, 0, 1)
    out["qsu_random_7_40_99_flat_4"] = {"state": hexs(st.view(np.float64)), "qr_log": log}
    psi = R.random_state(10, 4010)
    for p in (1, 4):
        e, nq, _ = R.expectation(psi, R.Terms.jw(10, 610), p, 0, 0, True, 1)
        out[f"evc_jw10_610_rs4010_p{p}"] = {"energy": [e.real, e.imag], "qr": nq}
    for n, golden in ((12, None), (16, None)):
        circ = R.Circuit.gatefabric(n, 4 * n, 1, True)
        terms = R.Terms.jw(n, 1, 0)
        for p in (1, 4):
            e, a, b = R.evaluate_energy(circ, terms, "flat", p, 0, 0, True, 1)
            out[f"energy_gf{n}_jw{n}_flat_p{p}"] = {"energy": e, "qsu_qr": a, "evc_qr": b}
    return out


def hea_arrays(n, depth):
    """Targets of gen_hea: per layer RY on every qubit, RZ on
    every qubit, CZ(q, q+1) for even q, then odd q.  Payload-free: only the
    targets matter to the schedulers."""
    ar, tg = [], []
    for _ in range(depth):
        for _ in range(2):
            for q in range(n):
                ar.append(1)
                tg.append(q)
        for parity in (0, 1):
            for q in range(parity, n - 1, 2):
                ar.append(2)
                tg += [q, q + 1]
    return np.array(ar, dtype=np.int32), np.array(tg, dtype=np.int32)


def hea_circuit(n, depth):
    import ctypes as C
    ar, tg = hea_arrays(n, depth)
    return R.Circuit(R.lib().ref_circuit_from_arrays(n, len(ar), ar.ctypes.data_as(C.POINTER(C.c_int)),
                                                     tg.ctypes.data_as(C.POINTER(C.c_int)), None))


def configs():
    """The BASELINE.json configs as the reference computes them:
    C1 energies + QR totals, C4 HEA schedules, C5 uniform-word plans."""
    out = {}
    # C1: 20q GateFabric layers 80 seed 1, full JW seed 1, flat(4), lazy vs eager
    circ = R.Circuit.gatefabric(20, 80, 1, True)
    terms = R.Terms.jw(20, 1, 0)
    for sched in ("flat", "adhoc"):
        e, a, b = R.evaluate_energy(circ, terms, sched, 4, 0, 0, True, 4)
        out[f"c1_{sched}"] = {"energy": e, "energy_hex": float(e).hex(), "qsu_qr": a, "evc_qr": b}
    # C4: HEA depth 20 schedules at 30/32/34 qubits
    hea = []
    for n in (20, 30, 32, 34):
        c = hea_circuit(n, 20)
        for p in (2, 4, 8):
            for sched in ("flat", "adhoc"):
                d = c.schedule(sched, p, 0, 0)
                hea.append({"circuit": f"hea:{n}:20", "shape": f"flat{p}", "scheduler": sched,
                            "counts": d["counts"], "tiles": len(d["schedule"]["tiles"]),
                            "sha": sha(d["schedule"]),
                            "events_sha": sha([e["after_pos_of"] for e in d["events"]])})
    out["hea_schedules"] = hea
    # C5 stress: 10,000 uniform words, Rng(2024)
    uni = []
    for n, count, p in ((34, 10000, 8), (34, 10000, 4), (34, 10000, 2), (32, 10000, 4), (30, 1000, 1), (30, 1000, 2)):
        t = R.Terms.uniform(n, count, 2024)
        letters, co = t.export()
        d = t.plan(n, p, 0, 0, True, 8)
        uni.append({"terms": f"uniform:{n}:{count}:2024", "shape": f"flat{p}", "diag": True,
                    "words_sha": hashlib.sha256("".join(letters).encode()).hexdigest(),
                    "coeff_sha": hashlib.sha256(co.tobytes()).hexdigest(),
                    "qr": d["qr_count"], "groups": d["n_groups"], "tiles": len(d["plan"]["tiles"]),
                    "sha": sha(d["plan"])})
    out["uniform_plans"] = uni
    # small-n uniform-word energies through the reference expectation (GPU parity)
    for n, count, p in ((16, 200, 1), (16, 200, 4), (18, 300, 2)):
        psi = R.random_state(n, 500 + n)
        e, nq, _ = R.expectation(psi, R.Terms.uniform(n, count, 2024), p, 0, 0, True, 4)
        out[f"evc_uniform_{n}_{count}_rs{500 + n}_p{p}"] = {"energy": [e.real, e.imag], "qr": nq}
    return out


def large():
    """Full iterations through the reference above the C1 size: 24 qubits (GateFabric layers 96
    seed 1, JW span-10, p = 8, lazy and eager; ~21 CPU-minutes with 8 workers) and 26 qubits
    (layers 104, lazy; ~45 CPU-minutes)."""
    out = {}
    circ = R.Circuit.gatefabric(24, 96, 1, True)
    terms = R.Terms.jw(24, 1, 10)
    for sched in ("flat", "adhoc"):
        e, a, b = R.evaluate_energy(circ, terms, sched, 8, 0, 0, True, 8)
        out[f"c24_{sched}_p8"] = {"energy": e, "energy_hex": float(e).hex(), "qsu_qr": a, "evc_qr": b}
    # 26 qubits, lazy only (~45 CPU-minutes with 8 workers)
    circ = R.Circuit.gatefabric(26, 104, 1, True)
    terms = R.Terms.jw(26, 1, 10)
    e, a, b = R.evaluate_energy(circ, terms, "flat", 8, 0, 0, True, 8)
    out["c26_flat_p8"] = {"energy": e, "energy_hex": float(e).hex(), "qsu_qr": a, "evc_qr": b}
    return out


def main():
    if not R.available():
        sys.exit("oracle/_ref/libqrtile_ref.so missing: run `make -C oracle ref` first")
    if sys.argv[1:] == ["large"]:  # merged into configs.json
        cfg = json.loads((HERE / "configs.json").read_text())
        cfg.update(large())
        (HERE / "configs.json").write_text(json.dumps(cfg, indent=0))
        return
    if sys.argv[1:] == ["configs"]:
        cfg = configs()
        old = HERE / "configs.json"
        if old.exists():  # keep the (slow) 24-qubit entries of `make_golden.py large`
            cfg.update({k: v for k, v in json.loads(old.read_text()).items() if k.startswith(("c24_", "c26_"))})
        (HERE / "configs.json").write_text(json.dumps(cfg, indent=0))
        return
    if not R.available():
        sys.exit("oracle/_ref/libqrtile_ref.so missing: run `make -C oracle ref` first")
    (HERE / "schedules.json").write_text(json.dumps(schedules(), indent=0))
    (HERE / "plans.json").write_text(json.dumps(plans(), indent=0))
    (HERE / "generators.json").write_text(json.dumps(generators(), indent=0))
    (HERE / "distsim.json").write_text(json.dumps(distsim(), indent=0))
    cfg = configs()
    old = HERE / "configs.json"
    if old.exists():  # keep the (slow) 24-qubit entries of `make_golden.py large`
        cfg.update({k: v for k, v in json.loads(old.read_text()).items() if k.startswith(("c24_", "c26_"))})
    (HERE / "configs.json").write_text(json.dumps(cfg, indent=0))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
