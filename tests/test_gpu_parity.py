"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Mirrors the reference's dist-sim unit tests (proj/tests/test_dist_sim.cpp) and
acceptance criteria (proj/tests/acceptance.cpp:81-173, 270-309).  Tolerances:
amplitudes within 1e-12 absolute on normalised states (the reference's own
bar, acceptance.cpp:113), energies within 1e-10 * (1 + |E|) (north_star:
1e-10 relative), QR moves bit-exact (a pure permutation).
"""
import numpy as np
import pytest

from oracle import cpu

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-12
E_TOL = 1e-10


def shape_for(qb, p):
    # acceptance.cpp:59-61
    return qb.ClusterShape.two_level(2, p // 2) if p >= 4 else qb.ClusterShape.flat(p)


def as_sub(state):
    return np.array(state.sub)


# ---------------------------------------------------------------- basics

def test_zero_state(qb, device):
    st = qb.init_state(2, qb.ClusterShape.flat(2))  # test_dist_sim.cpp:59-63
    sub = as_sub(st)
    assert sub[0].tolist() == [1.0, 0.0] and sub[1].tolist() == [0.0, 0.0]


def test_block_distribution(qb, device):
    amps = np.arange(16, dtype=np.complex128)  # test_dist_sim.cpp:65-75
    st = qb.init_state_from(amps, qb.ClusterShape.flat(4))
    sub = as_sub(st)
    for pe in range(4):
        assert sub[pe].real.tolist() == [pe * 4 + o for o in range(4)]
    assert np.array_equal(qb.flatten(st), amps)


def test_too_many_pes(qb, device):
    with pytest.raises(qb.TooManyPEs):
        qb.init_state(2, qb.ClusterShape.flat(4))


def test_x_gate_and_errors(qb, device):
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    st = qb.init_state(2, qb.ClusterShape.flat(2))
    qb.apply_gate_narrow(st, qb.make_gate(0, [0], X))
    sub = as_sub(st)
    assert sub[0][1] == 1.0 and sub[0][0] == 0.0
    st4 = qb.init_state(4, qb.ClusterShape.flat(4))
    with pytest.raises(qb.AccessViolation):
        qb.apply_gate_narrow(st4, qb.make_gate(0, [3], X))
    with pytest.raises(qb.MissingPayload):
        qb.apply_gate_narrow(st4, qb.make_gate(0, [0]))


def test_hadamard_twice_identity(qb, device):
    H = np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2)
    st = qb.init_state(4, qb.ClusterShape.flat(2))
    g = qb.make_gate(0, [0], H)
    qb.apply_gate_narrow(st, g)
    qb.apply_gate_narrow(st, g)
    f = qb.flatten(st)
    assert abs(f[0] - 1) <= 1e-15 and np.all(np.abs(f[1:]) <= 1e-15)


def test_cnot_convention(qb, device):
    # control = targets[0], flip targets[1] (test_dist_sim.cpp:33-41, 302-322)
    CNOT = np.zeros((4, 4), dtype=complex)
    CNOT[0, 0] = CNOT[2, 2] = CNOT[1, 3] = CNOT[3, 1] = 1
    X = np.array([[0, 1], [1, 0]], dtype=complex)
    st = qb.init_state(3, qb.ClusterShape.flat(1))
    qb.apply_gate_narrow(st, qb.make_gate(0, [2], X))
    qb.apply_gate_narrow(st, qb.make_gate(1, [2, 0], CNOT))
    f = qb.flatten(st)
    assert f[0b101] == 1.0


# ------------------------------------------------------- gates vs oracle

@pytest.mark.parametrize("n,p", [(8, 4), (13, 1), (16, 2), (18, 1)])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
def test_random_gate_matches_oracle(qb, device, n, p, k):
    rng = np.random.default_rng(1000 * n + 10 * p + k)
    nl = n - (p.bit_length() - 1)
    if k > nl:
        pytest.skip("gate wider than the local region")
    psi = qb.random_state(n, 7 + n)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(p))
    sub = psi.reshape(p, -1).copy()
    for trial in range(3):
        targets = [int(x) for x in rng.choice(nl, size=k, replace=False)]
        U = qb.random_unitary(k, int(rng.integers(1 << 62)))
        qb.apply_gate_narrow(st, qb.make_gate(trial, targets, U))
        cpu.apply_gate(sub, targets, U)
    err = np.max(np.abs(as_sub(st) - sub))
    assert err <= AMP_TOL, err


@pytest.mark.parametrize("n,p", [(10, 2), (15, 1), (20, 4)])
def test_diagonal_and_mixed_runs(qb, device, n, p):
    """RZ / CZ (diagonal fast path) interleaved with RY, many gates per call."""
    hea = qb.gen_hea(n, 3, 5)
    st = qb.init_state(n, qb.ClusterShape.flat(p))
    nl = n - (p.bit_length() - 1)
    ids = [op.id for op in hea.operators if all(q < nl for q in op.targets)]
    qb.apply_gates_narrow(st, hea, ids)
    sub = np.zeros((p, 1 << nl), dtype=complex)
    sub[0, 0] = 1
    for i in ids:
        op = hea.operators[i]
        cpu.apply_gate(sub, list(op.targets), op.payload)
    assert np.max(np.abs(as_sub(st) - sub)) <= AMP_TOL


def test_wide_gate_out_of_place(qb, device):
    """k = 9 exceeds the in-tile limit and takes the generic kernel."""
    n = 12
    psi = qb.random_state(n, 3)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(1))
    U = qb.random_unitary(9, 99)
    targets = [0, 2, 3, 5, 6, 7, 9, 10, 11]
    qb.apply_gate_narrow(st, qb.make_gate(0, targets, U))
    sub = psi.reshape(1, -1).copy()
    cpu.apply_gate(sub, targets, U)
    assert np.max(np.abs(as_sub(st) - sub)) <= AMP_TOL


# ------------------------------------------------------------------ QR

def test_qr_documented_pair(qb, device):
    # test_dist_sim.cpp:142-159: swap qubits 0 and 2 on n=4, p=4
    amps = np.arange(16, dtype=np.complex128)
    st = qb.init_state_from(amps, qb.ClusterShape.flat(4))
    ev = qb.make_qr_event(st.layout, 0b110)
    assert ev.swaps == [(0, 2)]
    moved = qb.perform_qr(st, ev)
    sub = as_sub(st)
    assert sub[1][0].real == 1.0 and sub[0][1].real == 4.0
    assert np.array_equal(qb.flatten(st), amps)
    assert moved == qb.qr_data_volume(1, 4)
    with pytest.raises(qb.LayoutMismatch):
        qb.perform_qr(st, ev)


@pytest.mark.parametrize("trial", range(12))
def test_qr_bit_exact_vs_oracle(qb, device, trial):
    rng = np.random.default_rng(77 + trial)
    n = int(rng.integers(4, 17))
    p = 1 << int(rng.integers(1, min(3, n - 1) + 1))
    psi = qb.random_state(n, 100 + trial)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(p))
    lay = cpu.Layout(n, p)
    sub = psi.reshape(p, -1).copy()
    for _ in range(3):
        locals_ = 0
        while bin(locals_).count("1") < st.n_local():
            locals_ |= 1 << int(rng.integers(n))
        ev = qb.make_qr_event(st.layout, locals_)
        if ev is None:
            continue
        moved = qb.perform_qr(st, ev)
        ref_moved = cpu.perform_qr(sub, lay.dest_for(ev.after.pos_of))
        lay.adopt(ev.after.pos_of)
        assert moved == ref_moved == qb.qr_data_volume(len(ev.swaps), n)
        assert np.array_equal(as_sub(st), sub)  # bit-exact
        assert np.array_equal(qb.flatten(st), psi)  # flatten invariant (acceptance.cpp:270-285)


# ------------------------------------------------------- QSU end to end

@pytest.mark.parametrize("sched", ["flat", "hierarchical", "adhoc"])
@pytest.mark.parametrize("n,p", [(12, 1), (12, 4), (16, 8), (18, 2)])
def test_run_qsu_gatefabric(qb, device, sched, n, p):
    c = qb.gen_gatefabric(n, 2 if n >= 16 else 4, 1, True)
    d = qb.build_dependency_graph(c)
    shape = shape_for(qb, p)
    s = {"flat": qb.flat_tiling, "hierarchical": qb.hierarchical_tiling, "adhoc": qb.adhoc_schedule}[sched](c, d, shape)
    st = qb.init_state(n, shape)
    qb.run_qsu(st, c, s)
    sub, lay, moved = cpu.run_qsu(n, p, c, s)
    got = qb.flatten(st)
    want = cpu.flatten(sub, lay.qubit_at)
    assert np.max(np.abs(got - want)) <= AMP_TOL
    assert [m for _, m in st.qr_log] == moved
    assert st.layout.pos_of == lay.pos_of


def test_random_circuits_acceptance(qb, device):
    """acceptance.cpp:81-126 on the GPU: seeded random circuits, every scheduler."""
    rng = np.random.default_rng(20241)
    worst = 0.0
    for case in range(30):
        n = int(rng.integers(4, 13))
        p = 1 << int(rng.integers(1, min(3, n - 2) + 1))
        m = int(rng.integers(1, 100))
        c = qb.gen_random_circuit(n, m, int(rng.integers(1 << 62)), 2, True)
        d = qb.build_dependency_graph(c)
        shape = shape_for(qb, p)
        for fn in (qb.flat_tiling, qb.hierarchical_tiling, qb.adhoc_schedule):
            s = fn(c, d, shape)
            st = qb.init_state(n, shape)
            qb.run_qsu(st, c, s)
            sub, lay, _ = cpu.run_qsu(n, p, c, s)
            worst = max(worst, float(np.max(np.abs(qb.flatten(st) - cpu.flatten(sub, lay.qubit_at)))))
            assert all(mv == qb.qr_data_volume(k, n) for k, mv in st.qr_log)
    assert worst <= AMP_TOL, worst


# ------------------------------------------------------------------ EVC

def oracle_expectation(qb, psi, n, p, terms, plan):
    """expectation() (dist_sim.cpp:263-300) on the C oracle, layout driven by
    make_qr_event from the product's (reference-identical) layouts."""
    sub = psi.reshape(p, -1).copy()
    lay = cpu.Layout(n, p)
    layout = qb.QubitLayout.identity(n, qb.ClusterShape.flat(p))
    partial = np.zeros(p, dtype=complex)
    for tile in plan.tiles:
        if layout.local_set() != tile.local_qubits:
            ev = qb.make_qr_event(layout, tile.local_qubits)
            if ev is not None:
                cpu.perform_qr(sub, lay.dest_for(ev.after.pos_of))
                lay.adopt(ev.after.pos_of)
                layout = ev.after
        masked = [cpu.mask_term(terms[i].letters, lay.pos_of, lay.nl) for i in tile.terms]
        partial += cpu.expectation_tile(sub, masked, [terms[i].coeff for i in tile.terms])
    return partial.sum()


@pytest.mark.parametrize("n", [8, 10, 12])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("diag", [True, False])
def test_expectation_jw(qb, device, n, p, diag):
    if p > (1 << (n - 2)):
        pytest.skip("p too large")
    terms = qb.gen_synthetic_jw(n, 600 + n) if (diag or p == 1) else qb.gen_synthetic_jw(n, 700 + n, n - 2)
    psi = qb.random_state(n, 4000 + n)
    shape = shape_for(qb, p)
    try:
        plan = qb.plan_evc(terms, n, shape, diag)
    except qb.TermTooWide:
        pytest.skip("terms do not tile without diagonalization")
    st = qb.init_state_from(psi, shape)
    got = qb.expectation(st, plan, terms)
    want = oracle_expectation(qb, psi, n, p, terms, plan)
    assert abs(got - want) <= E_TOL * (1 + abs(want))
    assert all(mv == qb.qr_data_volume(k, n) for k, mv in st.qr_log)


def test_expectation_basics(qb, device):
    # test_dist_sim.cpp:235-266: Z0 on |0> = +1, X0 on |+> = +1, global Z
    n = 4
    st = qb.init_state(n, qb.ClusterShape.flat(4))
    assert qb.diag_expectation_term(st, qb.PauliTerm(1.0, "ZIII")) == 1.0
    assert qb.diag_expectation_term(st, qb.PauliTerm(1.0, "IIIZ")) == 1.0
    H = np.array([[1, 1], [1, -1]], dtype=complex) / np.sqrt(2)
    qb.apply_gate_narrow(st, qb.make_gate(0, [0], H))
    assert abs(qb.diag_expectation_term(st, qb.PauliTerm(1.0, "XIII")) - 1.0) <= 1e-15
    with pytest.raises(qb.NotDiagonalizable):
        qb.diag_expectation_term(st, qb.PauliTerm(1.0, "IIIX"))


@pytest.mark.parametrize("n,golden", [(12, -0.94987699789824254), (16, -0.7881455344160232)])
def test_energy_golden(qb, device, n, golden):
    """GateFabric layers 4n seed 1, full JW seed 1."""
    c = qb.gen_gatefabric(n, 4 * n, 1, True)
    d = qb.build_dependency_graph(c)
    terms = qb.gen_synthetic_jw(n, 1)
    for p in (1, 2, 4, 8):
        shape = shape_for(qb, p)
        for fn in (qb.flat_tiling, qb.adhoc_schedule):
            s = fn(c, d, shape)
            plan = qb.plan_evc(terms, n, shape, True)
            e = qb.evaluate_energy(c, s, terms, plan)
            assert abs(e - golden) <= E_TOL * (1 + abs(golden)), (p, e)


# ------------------------------------------------ size-independent checks

def test_large_qr_roundtrip_and_norm(qb, device):
    """n=26 on 4 PEs: QR there and back is bit-exact; gates keep the norm."""
    n, p = 26, 4
    st = qb.init_state(n, qb.ClusterShape.flat(p))
    c = qb.gen_gatefabric(n, 2, 3, True)
    ids = [op.id for op in c.operators if all(q < n - 2 for q in op.targets)]
    qb.apply_gates_narrow(st, c, ids)
    before = [st.sub_of(pe) for pe in range(p)]
    locals0 = st.layout.local_set()  # st.layout is a live view; keep the value
    ev = qb.make_qr_event(st.layout, ((1 << n) - 1) & ~0b11)  # qubits 0,1 <-> 24,25
    qb.perform_qr(st, ev)
    assert st.last_relocated == qb.qr_data_volume(2, n)
    back = qb.make_qr_event(st.layout, locals0)
    qb.perform_qr(st, back)
    for pe in range(p):
        assert np.array_equal(st.sub_of(pe), before[pe])
    assert abs(st.norm() - 1.0) <= 1e-12


@pytest.mark.parametrize("n,p,k,linear", [(16, 1, 60, 1), (16, 2, 60, 1), (18, 4, 60, 1), (20, 1, 150, 1),
                                          (20, 2, 150, 1), (18, 2, 60, 0)])
def test_expectation_uniform_random_strings(qb, device, monkeypatch, n, p, k, linear):
    """Uniformly random words (SURVEY §8d C5 stress): most flip masks are wider
    than a shared-memory tile and take the GF(2)-linear passes (8 groups per
    HBM read); QRT_EVC_LINEAR=0 the full-vector sweeps (one per group)."""
    monkeypatch.setenv("QRT_EVC_LINEAR", str(linear))
    rng = np.random.default_rng(2024 + n + p + 100 * (1 - linear))  # distinct words: no plan-cache hit
    terms = []
    for _ in range(k):
        letters = "".join("IXYZ"[int(rng.integers(4))] for _ in range(n))
        # the 150-word cases use real coefficients (single-table Re(w) / Im(w) groups)
        im = 0.0 if k == 150 else rng.uniform(-0.1, 0.1)
        terms.append(qb.PauliTerm(complex(rng.uniform(-1, 1), im), letters))
    psi = qb.random_state(n, 77 + n)
    shape = qb.ClusterShape.flat(p)
    plan = qb.plan_evc(terms, n, shape, True, 4)
    st = qb.init_state_from(psi, shape)
    got = qb.expectation(st, plan, terms)
    want = oracle_expectation(qb, psi, n, p, terms, plan)
    assert abs(got - want) <= E_TOL * (1 + abs(want)), (got, want)


@pytest.mark.parametrize("k,diag,p,inplace", [(8, False, 1, "0"), (10, False, 2, "1"), (12, False, 1, "1"),
                                               (11, True, 2, "1"), (14, True, 1, "0")])
def test_wide_gate_in_place(qb, device, monkeypatch, k, diag, p, inplace):
    """Dense gates of 8..12 qubits run in place, one group of 2^k amplitudes
    per CTA (no spare buffer: also on single-buffer states); wide diagonals
    elementwise in place.  Checked against the oracle's apply_gate_narrow."""
    monkeypatch.setenv("QRT_QR_INPLACE", inplace)
    n = 16
    nl = n - (p.bit_length() - 1)
    rng = np.random.default_rng(k * 10 + p)
    psi = qb.random_state(n, 40 + k)
    st = qb.init_state_from(psi, qb.ClusterShape.flat(p))
    targets = [int(x) for x in rng.choice(nl, size=k, replace=False)]
    if diag:
        U = np.diag(np.exp(1j * rng.uniform(0, 6.28, size=1 << k)))
    else:  # dense and unitary, without a 2^k Gram-Schmidt on the host
        U = np.kron(qb.random_unitary(k - 6, int(rng.integers(1 << 40))), qb.random_unitary(6, int(rng.integers(1 << 40))))
    qb.apply_gate_narrow(st, qb.make_gate(0, targets, U))
    sub = psi.reshape(p, -1).copy()
    cpu.apply_gate(sub, targets, U)
    assert np.max(np.abs(as_sub(st) - sub)) <= AMP_TOL


def test_wide_gate_beyond_in_place_limit_single_buffer(qb, device, monkeypatch):
    """A dense 13-qubit gate needs the out-of-place kernel's second buffer: a
    single-buffer state reports it instead of failing silently."""
    monkeypatch.setenv("QRT_QR_INPLACE", "1")
    n = 16
    st = qb.init_state(n, qb.ClusterShape.flat(2))
    U = np.roll(np.eye(1 << 13, dtype=complex), 1, axis=0)  # a dense (non-diagonal) permutation
    with pytest.raises(qb.DeviceError):
        qb.apply_gate_narrow(st, qb.make_gate(0, list(range(13)), U))
