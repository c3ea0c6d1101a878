"""TEST INFRASTRUCTURE ONLY — ctypes face of the unmodified reference library
(oracle/_ref/libqrtile_ref.so, built from /root/reference/proj/src by
oracle/Makefile, see ref_shim.cpp).  ``available()`` is False where it was
never built; tests that need it skip, golden fixtures cover the rest.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

_SO = Path(__file__).resolve().parent / "_ref" / "libqrtile_ref.so"
_LIB = None


def available() -> bool:
    return _SO.exists()


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        L = C.CDLL(str(_SO))
        vp, P = C.c_void_p, C.POINTER
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [vp]
        for name, args in {
            "ref_circuit_gatefabric": [C.c_int, C.c_int, C.c_uint64, C.c_int],
            "ref_circuit_random": [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int],
            "ref_circuit_hea": [C.c_int, C.c_int, C.c_uint64],
            "ref_circuit_fixture": [C.c_char_p, C.c_uint64],
            "ref_circuit_from_arrays": [C.c_int, C.c_int, P(C.c_int), P(C.c_int), P(C.c_double)],
            "ref_terms_jw": [C.c_int, C.c_uint64, C.c_int],
            "ref_terms_fixture": [C.c_char_p],
            "ref_terms_uniform": [C.c_int, C.c_int, C.c_uint64],
            "ref_terms_from_arrays": [C.c_int, C.c_int, C.c_char_p, P(C.c_double)],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = vp
        for name in ["ref_circuit_free", "ref_terms_free"]:
            getattr(L, name).argtypes = [vp]
        for name in ["ref_circuit_n", "ref_circuit_m", "ref_circuit_total_targets", "ref_terms_count", "ref_terms_n"]:
            getattr(L, name).argtypes = [vp]
            getattr(L, name).restype = C.c_int
        L.ref_circuit_total_mat_doubles.argtypes = [vp]
        L.ref_circuit_total_mat_doubles.restype = C.c_int64
        L.ref_circuit_export.argtypes = [vp, P(C.c_int), P(C.c_int), P(C.c_double)]
        L.ref_terms_export.argtypes = [vp, C.c_char_p, P(C.c_double)]
        L.ref_schedule_json.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, C.c_int]
        L.ref_schedule_json.restype = vp
        L.ref_depth_sort_json.argtypes = [vp]
        L.ref_depth_sort_json.restype = vp
        L.ref_plan_json.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_plan_json.restype = vp
        L.ref_random_state.argtypes = [C.c_int, C.c_uint64, P(C.c_double)]
        L.ref_run_qsu.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_double),
                                  P(C.c_uint64), P(C.c_int), P(C.c_int)]
        L.ref_dense_qsu.argtypes = [vp, P(C.c_double)]
        L.ref_dense_expectation.argtypes = [P(C.c_double), C.c_int, vp, P(C.c_double)]
        L.ref_expectation.argtypes = [P(C.c_double), C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      P(C.c_double), P(C.c_int), P(C.c_double)]
        L.ref_evaluate_energy.argtypes = [vp, vp, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          P(C.c_double), P(C.c_int), P(C.c_int)]
        L.ref_time_prefix.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_double), P(C.c_double),
                                      P(C.c_double)]
        L.ref_time_sample.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_double), P(C.c_double)]
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError("reference: " + lib().ref_last_error().decode())


def _take_json(ptr) -> dict:
    if not ptr:
        raise RuntimeError("reference: " + lib().ref_last_error().decode())
    try:
        return json.loads(C.cast(ptr, C.c_char_p).value.decode())
    finally:
        lib().ref_free(ptr)


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Circuit:
    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference: " + lib().ref_last_error().decode())
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.ref_circuit_free(self.h)

    @classmethod
    def gatefabric(cls, n, layers, seed=1, payloads=True):
        return cls(lib().ref_circuit_gatefabric(n, layers, seed, int(payloads)))

    @classmethod
    def hea(cls, n, depth, seed=1):
        """SURVEY.md §8d C4 HEA built from reference types (ref_shim.cpp)."""
        return cls(lib().ref_circuit_hea(n, depth, seed))

    @property
    def m(self):
        return lib().ref_circuit_m(self.h)

    @classmethod
    def random(cls, n, m, seed, max_arity=2, payloads=True):
        return cls(lib().ref_circuit_random(n, m, seed, max_arity, int(payloads)))

    @classmethod
    def fixture(cls, name, seed=1):
        return cls(lib().ref_circuit_fixture(name.encode(), seed))

    @classmethod
    def from_product(cls, circ):
        """Mirror a product Circuit (targets + payloads) into the reference."""
        ar = np.array([op.arity() for op in circ.operators], dtype=np.int32)
        tg = np.array([q for op in circ.operators for q in op.targets], dtype=np.int32)
        pl = [op.payload for op in circ.operators]
        mats = None
        if all(x is not None for x in pl) and pl:
            mats = np.concatenate([np.ascontiguousarray(x, dtype=np.complex128).ravel() for x in pl]).view(np.float64)
        return cls(lib().ref_circuit_from_arrays(circ.n, len(ar), ar.ctypes.data_as(C.POINTER(C.c_int)),
                                                 tg.ctypes.data_as(C.POINTER(C.c_int)),
                                                 _d(mats) if mats is not None else None))

    @property
    def n(self):
        return lib().ref_circuit_n(self.h)

    def export(self):
        m = lib().ref_circuit_m(self.h)
        ar = np.zeros(m, dtype=np.int32)
        tg = np.zeros(lib().ref_circuit_total_targets(self.h), dtype=np.int32)
        nd = lib().ref_circuit_total_mat_doubles(self.h)
        mats = np.zeros(max(1, nd), dtype=np.float64)
        lib().ref_circuit_export(self.h, ar.ctypes.data_as(C.POINTER(C.c_int)), tg.ctypes.data_as(C.POINTER(C.c_int)),
                                 _d(mats) if nd else None)
        return ar, tg, mats[:nd]

    def schedule(self, name, p, n_node=0, n_gpn=0) -> dict:
        return _take_json(lib().ref_schedule_json(self.h, name.encode(), p, n_node, n_gpn))

    def depth_sort(self) -> dict:
        return _take_json(lib().ref_depth_sort_json(self.h))

    def run_qsu(self, sched, p, n_node=0, n_gpn=0, workers=1):
        n = self.n
        out = np.zeros(1 << n, dtype=np.complex128)
        moved = np.zeros(4096, dtype=np.uint64)
        ks = np.zeros(4096, dtype=np.int32)
        nq = C.c_int(0)
        _check(lib().ref_run_qsu(self.h, sched.encode(), p, n_node, n_gpn, workers, _d(out),
                                 moved.ctypes.data_as(C.POINTER(C.c_uint64)), ks.ctypes.data_as(C.POINTER(C.c_int)),
                                 C.byref(nq)))
        return out, list(zip(ks[:nq.value].tolist(), moved[:nq.value].tolist()))

    def dense(self):
        out = np.zeros(1 << self.n, dtype=np.complex128)
        _check(lib().ref_dense_qsu(self.h, _d(out)))
        return out


class Terms:
    @property
    def count(self):
        return lib().ref_terms_count(self.h)

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference: " + lib().ref_last_error().decode())
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.ref_terms_free(self.h)

    @classmethod
    def jw(cls, n, seed, max_span=0):
        return cls(lib().ref_terms_jw(n, seed, max_span))

    @classmethod
    def fixture(cls, name):
        return cls(lib().ref_terms_fixture(name.encode()))

    @classmethod
    def uniform(cls, n, count, seed=2024):
        return cls(lib().ref_terms_uniform(n, count, seed))

    @classmethod
    def from_product(cls, terms, n):
        letters = "".join(t.letters for t in terms).encode()
        co = np.array([t.coeff for t in terms], dtype=np.complex128)
        return cls(lib().ref_terms_from_arrays(n, len(terms), letters, _d(co)))

    def export(self):
        cnt, n = lib().ref_terms_count(self.h), lib().ref_terms_n(self.h)
        buf = C.create_string_buffer(cnt * n + 1)
        co = np.zeros(cnt, dtype=np.complex128)
        lib().ref_terms_export(self.h, buf, _d(co))
        raw = buf.raw[: cnt * n].decode()
        return [raw[i * n:(i + 1) * n] for i in range(cnt)], co

    def plan(self, n, p, n_node=0, n_gpn=0, diagonalize=True, workers=1) -> dict:
        return _take_json(lib().ref_plan_json(self.h, n, p, n_node, n_gpn, int(diagonalize), workers))


def random_state(n, seed):
    out = np.zeros(1 << n, dtype=np.complex128)
    _check(lib().ref_random_state(n, seed, _d(out)))
    return out


def expectation(canon, terms: Terms, p, n_node=0, n_gpn=0, diagonalize=True, workers=1):
    n = canon.size.bit_length() - 1
    out = np.zeros(2)
    nq = C.c_int(0)
    after = np.zeros_like(canon)
    _check(lib().ref_expectation(_d(np.ascontiguousarray(canon)), n, terms.h, p, n_node, n_gpn, int(diagonalize),
                                 workers, _d(out), C.byref(nq), _d(after)))
    return complex(out[0], out[1]), nq.value, after


def dense_expectation(canon, terms: Terms):
    n = canon.size.bit_length() - 1
    out = np.zeros(2)
    _check(lib().ref_dense_expectation(_d(np.ascontiguousarray(canon)), n, terms.h, _d(out)))
    return complex(out[0], out[1])


def evaluate_energy(circ: Circuit, terms: Terms, sched, p, n_node=0, n_gpn=0, diagonalize=True, workers=1):
    e = C.c_double(0)
    a, b = C.c_int(0), C.c_int(0)
    _check(lib().ref_evaluate_energy(circ.h, terms.h, sched.encode(), p, n_node, n_gpn, int(diagonalize), workers,
                                     C.byref(e), C.byref(a), C.byref(b)))
    return e.value, a.value, b.value


def time_sample(circ: Circuit, terms: Terms | None, p, workers, n_gates, n_terms):
    g, t = C.c_double(0), C.c_double(0)
    _check(lib().ref_time_sample(circ.h, terms.h if terms else None, p, workers, n_gates, n_terms, C.byref(g),
                                 C.byref(t)))
    return g.value, t.value


def time_prefix(circ: Circuit, terms: Terms | None, p, workers, per_arity=16, n_terms=64):
    """SURVEY.md §8d bounded sample: seconds per gate of each arity 1..4, per
    string, and per perform_qr of k = 1..log2 p (ref_shim.cpp ref_time_prefix)."""
    g = np.zeros(4)
    q = np.zeros(max(1, p.bit_length() - 1))
    t = C.c_double(0)
    _check(lib().ref_time_prefix(circ.h, terms.h if terms else None, p, workers, per_arity, n_terms, _d(g),
                                 C.byref(t), _d(q)))
    return g.tolist(), t.value, q.tolist()[: p.bit_length() - 1]
