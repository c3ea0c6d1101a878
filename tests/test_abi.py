"""The C-ABI library (CPU only: no compute calls without a GPU).

libqrt.so must load, export every entry point declared in include/qrt.h, and
fail loudly (QRT_ERR_NO_DEVICE + a message) when no device is present — the
product has no CPU fallback.
"""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "qrt.h").read_text()


def declared():
    names = re.findall(r"^\s*(?:qrt_status|const char\*|int)\s+(qrt_\w+)\s*\(", HEADER, flags=re.M)
    assert len(names) >= 15
    return names


def test_exports_every_declared_symbol(qb):
    lib = qb.load_libqrt()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_codes(qb):
    lib = qb.load_libqrt()
    assert lib.qrt_abi_version() == qb.QRT_ABI_VERSION == 2
    lib.qrt_last_error.restype = C.c_char_p
    assert isinstance(lib.qrt_last_error(), bytes)


def test_no_device_fails_loudly(qb):
    lib = qb.load_libqrt()
    n = C.c_int(-1)
    assert lib.qrt_device_count(C.byref(n)) == 0
    if n.value > 0:
        pytest.skip("a GPU is visible; covered by the gpu suite")
    st = C.c_void_p()
    rc = lib.qrt_state_create(4, 1, 0, None, C.byref(st))
    assert rc == 11  # QRT_ERR_NO_DEVICE
    lib.qrt_last_error.restype = C.c_char_p
    assert b"device" in lib.qrt_last_error()
    with pytest.raises(qb.DeviceError):
        qb.init_state(4, qb.ClusterShape.flat(1))


def test_argument_validation_without_device(qb):
    lib = qb.load_libqrt()
    st = C.c_void_p()
    assert lib.qrt_state_create(4, 3, 0, None, C.byref(st)) == 7  # QRT_ERR_CONFIG: p not a power of two
    assert lib.qrt_state_create(2, 8, 0, None, C.byref(st)) == 6  # QRT_ERR_TOO_MANY_PES
    assert lib.qrt_state_destroy(None) == 0


def test_native_libraries_are_in_tree(qb):
    pkg = Path(qb.__file__).parent
    for name in ("libqrt.so", "libqrtile_b200.so"):
        assert (pkg / name).exists()
    assert Path(qb._qrtile.__file__).parent == pkg


def _masks(terms):
    import numpy as np

    n = len(terms[0].letters)
    x = np.zeros(len(terms), np.uint64)
    y, z, gz = x.copy(), x.copy(), x.copy()
    co = np.zeros(2 * len(terms))
    for i, t in enumerate(terms):
        for q, c in enumerate(t.letters):
            bit = np.uint64(1 << q)
            if c == "X":
                x[i] |= bit
            elif c == "Y":
                y[i] |= bit
            elif c == "Z":
                z[i] |= bit
        co[2 * i], co[2 * i + 1] = t.coeff.real, t.coeff.imag
    return n, x, y, z, gz, co


def _plan_info(qb, terms):
    lib = qb.load_libqrt()
    n, x, y, z, gz, co = _masks(terms)
    P = C.POINTER(C.c_uint64)
    pa, gr, wi, sec = C.c_int(), C.c_int(), C.c_int(), C.c_double()
    rc = lib.qrt_pauli_plan_info(n, len(terms), x.ctypes.data_as(P), y.ctypes.data_as(P), z.ctypes.data_as(P),
                                 gz.ctypes.data_as(P), co.ctypes.data_as(C.POINTER(C.c_double)), C.byref(pa),
                                 C.byref(gr), C.byref(wi), C.byref(sec))
    assert rc == 0
    return pa.value, gr.value, wi.value, sec.value


def test_evc_pass_plan_host_only(qb):
    """EVC batching on the host (no device): 30-qubit JW span-10 packs 8,266
    strings into < 100 tile passes with no full-vector group, in milliseconds."""
    passes, groups, wide, sec = _plan_info(qb, qb.gen_synthetic_jw(30, 1, 10))
    assert 0 < passes < 100 and wide == 0 and groups >= 2000 and sec < 0.5
    import numpy as np

    rng = np.random.default_rng(1)
    rnd = [qb.PauliTerm(1.0, "".join("IXYZ"[int(v)] for v in rng.integers(0, 4, 30))) for _ in range(50)]
    passes_r, groups_r, wide_r, _ = _plan_info(qb, rnd)
    # random words: flip masks wider than a tile go to GF(2)-linear passes,
    # up to 10 groups per HBM read of the state, none to full-vector sweeps
    assert wide_r == 0 and groups_r == 50 and passes_r <= 7


def test_evc_linear_passes_knob(qb, monkeypatch):
    """QRT_EVC_LINEAR=0 restores one full-vector sweep per wide group."""
    import numpy as np

    rng = np.random.default_rng(3)
    rnd = [qb.PauliTerm(1.0, "".join("IXYZ"[int(v)] for v in rng.integers(0, 4, 28))) for _ in range(40)]
    monkeypatch.setenv("QRT_EVC_LINEAR", "0")
    _, _, wide_off, _ = _plan_info(qb, rnd)
    monkeypatch.setenv("QRT_EVC_LINEAR", "1")
    passes_on, _, wide_on, _ = _plan_info(qb, rnd)
    assert wide_off > 30 and wide_on == 0 and passes_on <= 6


def test_qr_bench_validation_without_device(qb):
    """qrt_qr_bench (single-process NVLink microbenchmark) rejects bad shapes
    before touching a device, and reports the missing GPUs loudly."""
    lib = qb.load_libqrt()
    ms, gbs = C.c_double(), C.c_double()
    assert lib.qrt_qr_bench(3, 28, 1, 1, 1, C.byref(ms), C.byref(gbs)) == 7   # QRT_ERR_CONFIG: not a power of two
    assert lib.qrt_qr_bench(2, 28, 2, 1, 1, C.byref(ms), C.byref(gbs)) == 7   # k > log2(n_gpus)
    assert lib.qrt_qr_bench(2, 8, 1, 1, 1, C.byref(ms), C.byref(gbs)) == 7    # n_local below a tile
    n = C.c_int(-1)
    lib.qrt_device_count(C.byref(n))
    if n.value < 2:
        assert lib.qrt_qr_bench(2, 28, 1, 1, 1, C.byref(ms), C.byref(gbs)) in (9, 11)  # CUDA / no device


def test_build_flags(qb):
    assert qb.build_flags() in (0, 1)
    chk = C.CDLL(str(Path(qb.__file__).parent / "libqrt_checked.so"))
    assert chk.qrt_build_flags() == 1 and qb.load_libqrt().qrt_build_flags() == 0
