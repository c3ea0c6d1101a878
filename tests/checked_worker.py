"""Runs under LD_PRELOAD=paper_2410_04252_b200/libqrt_checked.so (tests/test_gpu_checked.py):
the product's kernels with their device-side bounds and pipeline checks on,
over small cases covering every kernel family, each compared with the oracle.
A failed check traps the kernel, the call raises DeviceError and this exits 1."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2410_04252_b200 as qb  # noqa: E402
from oracle import cpu  # noqa: E402
from test_gpu_parity import oracle_expectation  # noqa: E402

assert qb.build_flags() & 1, "libqrt_checked.so is not the library in use"
qb.init_device(0, 1, 0)
cases = 0
for n, p, circ, sched, inplace in ((14, 4, "gf", "flat", "0"), (14, 2, "gf", "adhoc", "1"), (15, 8, "hea", "adhoc", "0"),
                                   (16, 1, "gf", "flat", "0"), (17, 2, "hea", "flat", "1")):
    os.environ["QRT_QR_INPLACE"] = inplace
    c = qb.gen_gatefabric(n, 2 * n, 3, True) if circ == "gf" else qb.gen_hea(n, 5, 3, True)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(p)
    s = (qb.flat_tiling if sched == "flat" else qb.adhoc_schedule)(c, d, shape)
    st = qb.init_state(n, shape)
    qb.run_qsu(st, c, s)
    sub, lay, _ = cpu.run_qsu(n, p, c, s)
    psi = cpu.flatten(sub, lay.qubit_at)
    assert float(np.max(np.abs(qb.flatten(st) - psi))) <= 1e-12, (n, p, circ)
    for terms in (qb.gen_synthetic_jw(n, 4, 10), qb.gen_uniform_words(n, 40, 2024)):
        try:
            plan = qb.plan_evc(terms, n, shape, True, 4)
        except qb.TermTooWide:  # uniform words wider than the local qubits at this p
            continue
        e = qb.expectation(qb.init_state_from(psi, shape), plan, terms)
        w = oracle_expectation(qb, psi, n, p, terms, plan)
        assert abs(e - w) <= 1e-10 * (1 + abs(w)), (n, p, circ, e, w)
        cases += 1
# a 20-qubit pipelined EVC (256 tiles per PE > one CTA per SM: every CTA walks several tiles)
n, p = 20, 2
psi = qb.random_state(n, 99)
for terms in (qb.gen_synthetic_jw(n, 6, 10), qb.gen_uniform_words(n, 200, 5)):
    plan = qb.plan_evc(terms, n, qb.ClusterShape.flat(p), True, 4)
    e = qb.expectation(qb.init_state_from(psi, qb.ClusterShape.flat(p)), plan, terms)
    w = oracle_expectation(qb, psi, n, p, terms, plan)
    assert abs(e - w) <= 1e-10 * (1 + abs(w)), (e, w)
    cases += 1
print("ok", cases)
