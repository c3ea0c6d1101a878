#!/usr/bin/env python
"""Gate-pass cost model: time one HBM pass holding G dense 4-qubit gates.

Every circuit's gates target 4-subsets of positions 0..11, so the planner puts
all G gates into one shared-memory pass; the pass time T(G) = a + b*G splits
into the per-pass cost a (tile load/store, setup) and the per-gate cost b
(DMMA work), which is compared with the DMMA-pipe floor.

  python tools/gate_sweep.py [--qubits 30] [--max-gates 8] [--reps 3]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2410_04252_b200 as qb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--max-gates", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n = args.qubits
    qb.init_device(0, 1, 0)
    rng = np.random.default_rng(7)
    shape = qb.ClusterShape.flat(1)
    st = qb.init_state(n, shape)
    st.profile(True)
    rows = []
    for G in range(1, args.max_gates + 1):
        ops = []
        for i in range(G):
            t = [int(x) for x in rng.choice(12, size=4, replace=False)]
            ops.append(qb.make_gate(i, t, qb.random_unitary(4, int(rng.integers(1 << 62)))))
        c = qb.Circuit(n, ops)
        sched = qb.flat_tiling(c, qb.build_dependency_graph(c), shape)
        best = None
        for _ in range(args.reps + 1):
            before = st.stats()["gates"]
            qb.run_qsu(st, c, sched)
            after = st.stats()["gates"]
            ms = after["ms"] - before["ms"]
            passes = after["launches"] - before["launches"]
            best = ms if best is None else min(best, ms)
        rows.append({"gates": G, "passes": passes, "ms": best})
        print(json.dumps(rows[-1]), flush=True)
    g = np.array([r["gates"] for r in rows], float)
    t = np.array([r["ms"] for r in rows], float)
    b, a = np.polyfit(g, t, 1)
    # DMMA floor per gate: 2^n/128 DMMA.8x8x4 (Gauss form: 24 per 8 groups of 16) x 16 cycles / (4 SMSP x SMs)
    print(json.dumps({"fit_ms_per_pass": a, "fit_ms_per_gate": b}))


if __name__ == "__main__":
    main()
