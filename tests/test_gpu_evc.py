"""GPU parity of the register-coset EVC kernel (csrc/qrt_coset.cu).

expectation() (dist_sim.cpp:263-300) on states whose local region holds a
full 2^12-amplitude tile, so flip-mask groups of <= 5 positions take the
coset path: Jordan-Wigner words (Re-only, real coefficients) and random
low-weight words with complex coefficients, odd Y counts and global Z letters
(the general table mode).  Checked against the C oracle and against the
shared-memory pair kernel (QRT_EVC_COSET=0).  Tolerance: 1e-10 (1 + |E|).
"""
import numpy as np
import pytest

from test_gpu_parity import oracle_expectation

pytestmark = pytest.mark.gpu

E_TOL = 1e-10


def _random_words(qb, rng, n, count, span, weight):
    terms = []
    for _ in range(count):
        start = int(rng.integers(0, n - span + 1))
        k = int(rng.integers(1, weight + 1))
        qs = rng.choice(np.arange(start, start + span), size=k, replace=False)
        letters = ["I"] * n
        for q in qs:
            letters[int(q)] = "XYZ"[int(rng.integers(3))]
        # occasional Z string far away (global positions at p > 1)
        if rng.random() < 0.3:
            letters[n - 1] = "Z" if letters[n - 1] == "I" else letters[n - 1]
        terms.append(qb.PauliTerm(complex(rng.uniform(-1, 1), rng.uniform(-0.5, 0.5)), "".join(letters)))
    return terms


@pytest.mark.parametrize("n,p,span", [(14, 1, 10), (16, 1, 10), (18, 2, 8), (20, 4, 10), (17, 8, 6)])
def test_coset_jw_vs_oracle(qb, device, n, p, span):
    terms = qb.gen_synthetic_jw(n, 31 + n, span)
    psi = qb.random_state(n, 900 + n)
    shape = qb.ClusterShape.flat(p)
    plan = qb.plan_evc(terms, n, shape, True)
    st = qb.init_state_from(psi, shape)
    got = qb.expectation(st, plan, terms)
    want = oracle_expectation(qb, psi, n, p, terms, plan)
    assert abs(got - want) <= E_TOL * (1 + abs(want)), (got, want)


@pytest.mark.parametrize("n,p", [(15, 1), (16, 2), (18, 4)])
def test_coset_general_words_vs_oracle(qb, device, n, p):
    rng = np.random.default_rng(7 * n + p)
    terms = _random_words(qb, rng, n, 300, 9, 5)
    psi = qb.random_state(n, 321 + n)
    shape = qb.ClusterShape.flat(p)
    plan = qb.plan_evc(terms, n, shape, True, 4)
    st = qb.init_state_from(psi, shape)
    got = qb.expectation(st, plan, terms)
    want = oracle_expectation(qb, psi, n, p, terms, plan)
    assert abs(got - want) <= E_TOL * (1 + abs(want)), (got, want)


def test_coset_matches_pair_kernel(qb, device, monkeypatch):
    """Same energy (to rounding) with the coset path on and off."""
    n = 19
    terms = qb.gen_synthetic_jw(n, 5, 10)
    psi = qb.random_state(n, 77)
    shape = qb.ClusterShape.flat(2)
    plan = qb.plan_evc(terms, n, shape, True)
    vals = {}
    for on in ("1", "0"):
        monkeypatch.setenv("QRT_EVC_COSET", on)
        st = qb.init_state_from(psi, shape)
        vals[on] = qb.expectation(st, plan, terms)
    assert abs(vals["1"] - vals["0"]) <= 1e-12 * (1 + abs(vals["0"]))


def test_coset_deterministic(qb, device):
    """Fixed reduction order: bit-identical energies run to run."""
    n = 18
    terms = qb.gen_synthetic_jw(n, 2, 10)
    psi = qb.random_state(n, 5)
    shape = qb.ClusterShape.flat(1)
    plan = qb.plan_evc(terms, n, shape, True)
    e = [qb.expectation(qb.init_state_from(psi, shape), plan, terms) for _ in range(3)]
    assert e[0] == e[1] == e[2]


@pytest.mark.parametrize("env", [{"QRT_EVC_GLOBAL_COVER": "0"}, {"QRT_COSET_OCC": "3"}, {"QRT_GATE_THREADS": "64"},
                                 {"QRT_PLAN_CACHE": "0"}, {"QRT_GAUSS": "0"}, {"QRT_GAUSS": "1"}, {"QRT_GATE_REGS": "128"},
                                 {"QRT_EVC_LINEAR": "0"}, {"QRT_EVC_PIPE": "0"}, {"QRT_EVC_SPLIT": "1"},
                                 {"QRT_QR_PUSH": "1", "QRT_FUSED_QR": "0", "QRT_QR_INPLACE": "0"},
                                 {"QRT_FUSED_QR": "0"}, {"QRT_EVC_SET_TABLES": "0"}, {"QRT_EVC_PRESENT_GUARD": "0"},
                                 {"QRT_EVC_FILL": "1"}, {"QRT_EVC_TEAMS": "1"}, {"QRT_EVC_PLAN_BATCHED": "0"},
                                 {"QRT_EVC_LINEAR_COAL": "3"}, {"QRT_EVC_SINGLE": "0"}])
def test_knobs_in_subprocess(env):
    """Knobs read once per process: a fresh process per setting, checked
    against the oracle (GateFabric QSU + JW EVC at 16 qubits, 2 PEs)."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, sys\n"
        "sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "import paper_2410_04252_b200 as qb\n"
        "from oracle import cpu\n"
        "from test_gpu_parity import oracle_expectation\n"
        "qb.init_device(0, 1, 0)\n"
        "n, p = 16, 2\n"
        "c = qb.gen_gatefabric(n, 8, 2, True)\n"
        "shape = qb.ClusterShape.flat(p)\n"
        "s = qb.flat_tiling(c, qb.build_dependency_graph(c), shape)\n"
        "st = qb.init_state(n, shape); qb.run_qsu(st, c, s)\n"
        "sub, lay, _ = cpu.run_qsu(n, p, c, s)\n"
        "psi = cpu.flatten(sub, lay.qubit_at)\n"
        "assert float(np.max(np.abs(qb.flatten(st) - psi))) <= 1e-12\n"
        "terms = qb.gen_synthetic_jw(n, 3, 10)\n"
        "plan = qb.plan_evc(terms, n, shape, True)\n"
        "e = qb.expectation(qb.init_state_from(psi, shape), plan, terms)\n"
        "w = oracle_expectation(qb, psi, n, p, terms, plan)\n"
        "assert abs(e - w) <= 1e-10 * (1 + abs(w)), (e, w)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=root, capture_output=True,
                         text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
