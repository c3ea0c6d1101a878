"""Uniform-word (C5 stress) energy vs p on one GPU against the C oracle at p = 1:
the reproducer of the round-1 EVC pipeline race (profiles/r2/uniform24_race_repro.txt).
  python tools/uniform_cross_p.py N COUNT P1,P2,... [nooracle]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2410_04252_b200 as qb  # noqa: E402
from oracle import cpu  # noqa: E402

n, count = int(sys.argv[1]), int(sys.argv[2])
ps = [int(x) for x in sys.argv[3].split(",")]
qb.init_device(0, 1, 0)
terms = qb.gen_uniform_words(n, count, 2024)
psi = qb.random_state(n, 1234)
if len(sys.argv) > 4 and sys.argv[4] == "nooracle":
    want = 0j
else:
    masked = [cpu.mask_term(t.letters, list(range(n)), n) for t in terms]
    want = cpu.expectation_tile(psi.reshape(1, -1).copy(), masked, [t.coeff for t in terms]).sum()
out = {"n": n, "count": count, "oracle": want.real}
for p in ps:
    shape = qb.ClusterShape.flat(p)
    plan = qb.plan_evc(terms, n, shape, True, 8)
    st = qb.init_state_from(psi, shape)
    e = qb.expectation(st, plan, terms)
    out[f"p{p}"] = [e.real, abs(e - want), len(plan.tiles)]
print(json.dumps(out))
