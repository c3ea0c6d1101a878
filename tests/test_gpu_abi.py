"""Parity through the raw C ABI (include/qrt.h) via ctypes — the binding a
reference caller would add — against the C oracle."""
import ctypes as C

import numpy as np
import pytest

from oracle import cpu

pytestmark = pytest.mark.gpu


def _lib(qb):
    lib = qb.load_libqrt()
    lib.qrt_last_error.restype = C.c_char_p
    return lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def test_abi_gates_qr_expectation(qb, device):
    lib = _lib(qb)
    n, p = 14, 4
    nl = n - 2
    rng = np.random.default_rng(3)
    psi = qb.random_state(n, 21).reshape(p, -1).copy()
    st = C.c_void_p()
    assert lib.qrt_state_create(n, p, 0, None, C.byref(st)) == 0, lib.qrt_last_error()
    try:
        for pe in range(p):
            assert lib.qrt_state_upload(st, pe, _d(np.ascontiguousarray(psi[pe]))) == 0
        # a batch of mixed gates through one call
        arity, pos, mats, flags = [], [], [], []
        ref = psi.copy()
        for g in range(12):
            k = int(rng.integers(1, 5))
            t = [int(x) for x in rng.choice(nl, size=k, replace=False)]
            diag = g % 3 == 0
            if diag:
                d = np.exp(1j * rng.uniform(0, 6.28, size=1 << k))
                u = np.diag(d)
                mats.append(d)
            else:
                u = qb.random_unitary(k, int(rng.integers(1 << 40)))
                mats.append(u.ravel())
            arity.append(k)
            pos.extend(t)
            flags.append(1 if diag else 0)
            cpu.apply_gate(ref, t, u)
        m = np.ascontiguousarray(np.concatenate(mats))
        rc = lib.qrt_apply_gates(st, len(arity), (C.c_int * len(arity))(*arity), (C.c_int * len(pos))(*pos), _d(m),
                                 (C.c_uint * len(flags))(*flags))
        assert rc == 0, lib.qrt_last_error()
        # a QR swapping positions 0,5 <-> 12,13 (both global bits)
        dest = list(range(n))
        dest[0], dest[12] = 12, 0
        dest[5], dest[13] = 13, 5
        moved = C.c_uint64()
        assert lib.qrt_reorder(st, (C.c_int * n)(*dest), C.byref(moved)) == 0, lib.qrt_last_error()
        ref_moved = cpu.perform_qr(ref, dest)
        assert moved.value == ref_moved == (1 << n) - (1 << (n - 2))
        got = np.empty((p, 1 << nl), dtype=np.complex128)
        for pe in range(p):
            assert lib.qrt_state_download(st, pe, _d(got[pe])) == 0
        assert np.max(np.abs(got - ref)) <= 1e-12
        # two Pauli words in position space: X0 Z1 Y7 with a global Z on PE bit 1, and Z3
        x = (C.c_uint64 * 2)(1, 0)
        y = (C.c_uint64 * 2)(1 << 7, 0)
        z = (C.c_uint64 * 2)(1 << 1, 1 << 3)
        gz = (C.c_uint64 * 2)(2, 0)
        co = np.array([0.7 + 0.1j, -0.3], dtype=np.complex128)
        partial = np.zeros(2 * p)
        assert lib.qrt_pauli_expectation(st, 2, x, y, z, gz, _d(co), _d(partial)) == 0, lib.qrt_last_error()
        terms = [cpu.MaskedTerm(1, 1 << 7, 1 << 1, 2, 1), cpu.MaskedTerm(0, 0, 1 << 3, 0, 0)]
        want = cpu.expectation_tile(ref, terms, co)
        assert np.max(np.abs(partial.view(np.complex128) - want)) <= 1e-12
        # errors surface as status codes + message
        bad = (C.c_int * 1)(nl)  # a global position
        assert lib.qrt_apply_gates(st, 1, (C.c_int * 1)(1), bad, _d(np.eye(2, dtype=complex).ravel()), None) == 2
        assert b"global" in lib.qrt_last_error()
    finally:
        assert lib.qrt_state_destroy(st) == 0


@pytest.mark.parametrize("kind", ["jw", "uniform"])
def test_abi_per_pe_partials_pipelined(qb, device, kind):
    """Per-PE partials (dist_sim.cpp:289-295) from the persistent pipelined
    EVC kernels: 2^20 amplitudes per PE = 256 tiles, more than one CTA per SM
    covers, so every CTA walks several tiles and the slot layout matters."""
    lib = _lib(qb)
    n, p = 22, 4
    nl = n - 2
    psi = qb.random_state(n, 2024).reshape(p, -1).copy()
    if kind == "jw":
        words = [t for t in qb.gen_synthetic_jw(nl, 5, 6) if set(t.letters) & {"X", "Y"}][:300]
    else:
        words = qb.gen_uniform_words(nl, 120, 7)
    x, y, z, co = [], [], [], []
    rng = np.random.default_rng(1)
    for t in words:
        xm = sum(1 << q for q, ch in enumerate(t.letters) if ch == "X")
        ym = sum(1 << q for q, ch in enumerate(t.letters) if ch == "Y")
        zm = sum(1 << q for q, ch in enumerate(t.letters) if ch == "Z")
        if xm | ym == 0:
            continue
        x.append(xm), y.append(ym), z.append(zm), co.append(t.coeff)
    m = len(x)
    gz = [int(rng.integers(0, p)) for _ in range(m)]
    co = np.array(co, dtype=np.complex128)
    st = C.c_void_p()
    assert lib.qrt_state_create(n, p, 0, None, C.byref(st)) == 0, lib.qrt_last_error()
    try:
        for pe in range(p):
            assert lib.qrt_state_upload(st, pe, _d(np.ascontiguousarray(psi[pe]))) == 0
        U = C.c_uint64 * m
        partial = np.zeros(2 * p)
        assert lib.qrt_pauli_expectation(st, m, U(*x), U(*y), U(*z), U(*gz), _d(co), _d(partial)) == 0, \
            lib.qrt_last_error()
        terms = [cpu.MaskedTerm(x[i], y[i], z[i], gz[i], bin(y[i]).count("1")) for i in range(m)]
        want = cpu.expectation_tile(psi, terms, co)
        assert np.max(np.abs(partial.view(np.complex128) - want)) <= 1e-12 * (1 + np.max(np.abs(want)))
    finally:
        assert lib.qrt_state_destroy(st) == 0
