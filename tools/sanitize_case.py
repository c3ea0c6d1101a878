"""Small VQE iterations for compute-sanitizer (racecheck / synccheck / memcheck):
covers the fused-QR gate passes (p = 4 on one GPU), the light passes (HEA),
the register-coset EVC kernels incl. the persistent pipelines (JW, split and
unsplit) and the linear passes (uniform words), and the in-place QR."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_2410_04252_b200 as qb  # noqa: E402

qb.init_device(0, 1, 0)
out = []
for n, p, circ in ((14, 4, "gf"), (15, 2, "hea"), (16, 1, "gf")):
    c = qb.gen_gatefabric(n, 2 * n, 1, True) if circ == "gf" else qb.gen_hea(n, 4, 1, True)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(p)
    s = qb.flat_tiling(c, d, shape)
    for terms in (qb.gen_synthetic_jw(n, 1, 8), qb.gen_uniform_words(n, 64, 2024)):
        plan = qb.plan_evc(terms, n, shape, True, 4)
        st = qb.init_state(n, shape)
        qb.run_qsu(st, c, s)
        e = qb.expectation(st, plan, terms)
        out.append((n, p, circ, len(terms), e.real, len(st.qr_log)))
        del st
os.environ["QRT_QR_INPLACE"] = "1"
st = qb.init_state(14, qb.ClusterShape.flat(4))
c = qb.gen_gatefabric(14, 28, 2, True)
qb.run_qsu(st, c, qb.adhoc_schedule(c, qb.build_dependency_graph(c), qb.ClusterShape.flat(4)))
out.append(("inplace", abs(st.norm() - 1.0) < 1e-12, len(st.qr_log)))
for o in out:
    print(o)
