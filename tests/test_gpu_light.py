"""GPU parity of the register-resident light gate passes (csrc/qrt_light.cu).

Runs of 1-/2-qubit dense gates and diagonal gates (phases and +-1 signs) —
the hardware-efficient-ansatz shape of BASELINE config C4 — applied through
apply_gates_narrow / run_qsu (reference apply_gate_narrow, dist_sim.cpp:163-201,
run_qsu :242-252) and compared with the CPU oracle gate by gate.  Local regions
of >= 12 positions take the light kernel; the planner fuses single-qubit
chains on the host (QRT_FUSE_1Q) and cuts passes into register stages
(QRT_LIGHT_STAGES); both are exercised against the unfused / heavy path too.
Tolerance: 1e-12 absolute on normalised states (acceptance.cpp:113).
"""
import os

import numpy as np
import pytest

from oracle import cpu

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-12


def _sub(st):
    return np.array(st.sub)


def _random_light_ops(qb, rng, nl, count):
    """Mixed 1q dense, 2q dense, 1-/2-qubit phase diagonals, +-1 sign
    diagonals up to 6 qubits, plus the odd 3-qubit phase diagonal (heavy)."""
    ops = []
    for i in range(count):
        r = rng.random()
        if r < 0.35:
            k, U = 1, qb.random_unitary(1, int(rng.integers(1 << 62)))
        elif r < 0.5:
            k, U = 2, qb.random_unitary(2, int(rng.integers(1 << 62)))
        elif r < 0.65:
            k = int(rng.integers(1, 3))
            U = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, size=1 << k)))
        elif r < 0.95:
            k = int(rng.integers(1, 7))
            d = np.where(rng.random(1 << k) < 0.5, -1.0, 1.0).astype(complex)
            U = np.diag(d)
        else:
            k = 3
            U = np.diag(np.exp(1j * rng.uniform(0, 2 * np.pi, size=8)))
        # bias targets towards the low (coalescing) and high positions
        pool = list(range(min(nl, 6))) + list(range(nl - 6, nl)) + list(range(nl))
        targets = []
        while len(targets) < k:
            q = int(pool[int(rng.integers(len(pool)))])
            if q not in targets:
                targets.append(q)
        ops.append(qb.make_gate(i, targets, U))
    return ops


@pytest.mark.parametrize("n,p,count,seed", [(12, 1, 120, 1), (14, 1, 300, 2), (16, 2, 400, 3),
                                            (18, 4, 400, 4), (20, 1, 250, 5), (13, 2, 200, 6)])
def test_light_random_runs_vs_oracle(qb, device, n, p, count, seed):
    rng = np.random.default_rng(seed)
    nl = n - (p.bit_length() - 1)
    ops = _random_light_ops(qb, rng, nl, count)
    circ = qb.Circuit(n, ops)
    psi = qb.random_state(n, 50 + seed)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(p))
    qb.apply_gates_narrow(st, circ, list(range(count)))
    sub = psi.reshape(p, -1).copy()
    for op in ops:
        cpu.apply_gate(sub, list(op.targets), op.payload)
    err = float(np.max(np.abs(_sub(st) - sub)))
    assert err <= AMP_TOL, err


@pytest.mark.parametrize("stages", ["1", "2", "8"])
@pytest.mark.parametrize("fuse", ["0", "1"])
def test_light_stage_and_fusion_knobs(qb, device, stages, fuse, monkeypatch):
    """QRT_FUSE_1Q / QRT_PHASE_FOLD are read per call; QRT_LIGHT_STAGES once per
    process, so the stage counts here run in a subprocess."""
    if stages != "1":
        import subprocess
        import sys
        code = (
            "import numpy as np, sys\n"
            "sys.path.insert(0, '.')\n"
            "import paper_2410_04252_b200 as qb\n"
            "from oracle import cpu\n"
            "qb.init_device(0, 1, 0)\n"
            "n = 16\n"
            "c = qb.gen_hea(n, 6, 9, True)\n"
            "st = qb.init_state(n, qb.ClusterShape.flat(1))\n"
            "qb.apply_gates_narrow(st, c, list(range(c.size())))\n"
            "sub = np.zeros((1, 1 << n), dtype=complex); sub[0, 0] = 1\n"
            "for op in c.operators: cpu.apply_gate(sub, list(op.targets), op.payload)\n"
            "err = float(np.max(np.abs(np.array(st.sub) - sub)))\n"
            "assert err <= 1e-12, err\n"
            "print('ok', err)\n")
        env = dict(os.environ, QRT_LIGHT_STAGES=stages, QRT_FUSE_1Q=fuse)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        res = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                             timeout=300)
        assert res.returncode == 0, res.stdout + res.stderr
        return
    monkeypatch.setenv("QRT_FUSE_1Q", fuse)
    monkeypatch.setenv("QRT_PHASE_FOLD", fuse)  # row-phase folding on/off with fusion
    n = 15
    c = qb.gen_hea(n, 5, 11, True)
    st = qb.init_state(n, qb.ClusterShape.flat(1))
    qb.apply_gates_narrow(st, c, list(range(c.size())))
    sub = np.zeros((1, 1 << n), dtype=complex)
    sub[0, 0] = 1
    for op in c.operators:
        cpu.apply_gate(sub, list(op.targets), op.payload)
    assert float(np.max(np.abs(_sub(st) - sub))) <= AMP_TOL


def test_light_matches_heavy_path(qb, device, monkeypatch):
    """The light kernel and the shared-memory gate kernel agree on an HEA run."""
    n = 17
    c = qb.gen_hea(n, 8, 21, True)
    ids = list(range(c.size()))
    out = {}
    for light in ("1", "0"):
        monkeypatch.setenv("QRT_LIGHT", light)
        st = qb.init_state(n, qb.ClusterShape.flat(2))
        qb.apply_gates_narrow(st, c, [i for i in ids if all(q < n - 1 for q in c.operators[i].targets)])
        out[light] = _sub(st)
    assert float(np.max(np.abs(out["1"] - out["0"]))) <= AMP_TOL


@pytest.mark.parametrize("sched", ["flat", "adhoc"])
@pytest.mark.parametrize("n,p,depth", [(16, 1, 10), (18, 4, 6), (20, 2, 4), (16, 8, 8)])
def test_run_qsu_hea_vs_oracle(qb, device, sched, n, p, depth):
    """C4's circuit family end to end: lazy / eager schedules, QRs included."""
    c = qb.gen_hea(n, depth, 1, True)
    d = qb.build_dependency_graph(c)
    shape = qb.ClusterShape.flat(p)
    s = (qb.flat_tiling if sched == "flat" else qb.adhoc_schedule)(c, d, shape)
    st = qb.init_state(n, shape)
    qb.run_qsu(st, c, s)
    sub, lay, moved = cpu.run_qsu(n, p, c, s)
    got = qb.flatten(st)
    want = cpu.flatten(sub, lay.qubit_at)
    assert float(np.max(np.abs(got - want))) <= AMP_TOL
    assert [m for _, m in st.qr_log] == moved
    assert abs(st.norm() - 1.0) <= 1e-12


def test_light_pass_count_and_launches(qb, device):
    """HEA at 20 qubits: the light planner needs far fewer HBM passes than gates."""
    n = 20
    c = qb.gen_hea(n, 20, 1, True)
    st = qb.init_state(n, qb.ClusterShape.flat(1))
    st.reset_stats()
    qb.apply_gates_narrow(st, c, list(range(c.size())))
    g = st.stats()["gates"]
    assert 0 < g["launches"] <= c.size() // 8, g


@pytest.mark.parametrize("merge", ["0", "1"])
def test_light_sign_merging(qb, device, merge, monkeypatch):
    """CZ/CCZ-heavy runs with sign-op pooling on and off (QRT_MERGE_SIGNS)."""
    monkeypatch.setenv("QRT_MERGE_SIGNS", merge)
    rng = np.random.default_rng(404)
    n, p = 17, 2
    nl = n - 1
    ops = []
    for i in range(500):
        if rng.random() < 0.25:
            ops.append(qb.make_gate(i, [int(rng.integers(nl))], qb.random_unitary(1, int(rng.integers(1 << 62)))))
        else:
            k = int(rng.integers(1, 4))
            targets = [int(x) for x in rng.choice(nl, size=k, replace=False)]
            d = np.ones(1 << k, dtype=complex)
            d[-1] = -1  # CZ / CCZ / Z
            ops.append(qb.make_gate(i, targets, np.diag(d)))
    circ = qb.Circuit(n, ops)
    psi = qb.random_state(n, 404)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(p))
    qb.apply_gates_narrow(st, circ, list(range(len(ops))))
    sub = psi.reshape(p, -1).copy()
    for op in ops:
        cpu.apply_gate(sub, list(op.targets), op.payload)
    assert float(np.max(np.abs(_sub(st) - sub))) <= AMP_TOL


def test_plan_cache_repacks_new_angles(qb, device):
    """A VQE loop: same circuit structure, new angles every iteration.  The
    cached pass decomposition must be re-packed with the new payloads."""
    n = 16
    for seed in (3, 4, 3, 5):
        c = qb.gen_hea(n, 6, seed, True)
        st = qb.init_state(n, qb.ClusterShape.flat(1))
        qb.apply_gates_narrow(st, c, list(range(c.size())))
        sub = np.zeros((1, 1 << n), dtype=complex)
        sub[0, 0] = 1
        for op in c.operators:
            cpu.apply_gate(sub, list(op.targets), op.payload)
        assert float(np.max(np.abs(_sub(st) - sub))) <= AMP_TOL, seed
    for seed in (7, 8):  # GateFabric (DMMA fragments re-packed)
        c = qb.gen_gatefabric(14, 8, seed, True)
        st = qb.init_state(14, qb.ClusterShape.flat(1))
        qb.apply_gates_narrow(st, c, list(range(c.size())))
        sub = np.zeros((1, 1 << 14), dtype=complex)
        sub[0, 0] = 1
        for op in c.operators:
            cpu.apply_gate(sub, list(op.targets), op.payload)
        assert float(np.max(np.abs(_sub(st) - sub))) <= AMP_TOL, seed
