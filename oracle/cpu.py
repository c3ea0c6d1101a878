"""TEST INFRASTRUCTURE ONLY — ctypes face of the C restatement (qrt_oracle.c).

State convention: a complex128 numpy array of shape (p, 2^nl), PE-major, the
reference's ``DistributedState::sub`` (dist_sim.hpp:28-41).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None


class MaskedTerm(C.Structure):
    _fields_ = [("x", C.c_uint64), ("y", C.c_uint64), ("z", C.c_uint64), ("global_z", C.c_uint64),
                ("y_count", C.c_int)]


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        so = _HERE / "liboracle.so"
        src = _HERE / "qrt_oracle.c"
        if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
            subprocess.run(["make", "-s", "-C", str(_HERE), "oracle"], check=True)
        L = C.CDLL(str(so))
        P = C.POINTER
        L.orc_apply_gate.argtypes = [P(C.c_double), C.c_int, C.c_int, C.c_int, P(C.c_int), P(C.c_double)]
        L.orc_perform_qr.argtypes = [P(C.c_double), P(C.c_double), C.c_int, C.c_int, C.c_int, P(C.c_int)]
        L.orc_perform_qr.restype = C.c_uint64
        L.orc_mask_term.argtypes = [C.c_char_p, C.c_int, P(C.c_int), C.c_int, P(MaskedTerm)]
        L.orc_local_pauli.argtypes = [P(C.c_double), C.c_uint64, P(MaskedTerm), P(C.c_double)]
        L.orc_expectation_tile.argtypes = [P(C.c_double), C.c_int, C.c_int, C.c_int, P(MaskedTerm),
                                           P(C.c_double), P(C.c_double)]
        L.orc_flatten.argtypes = [P(C.c_double), C.c_int, C.c_int, C.c_int, P(C.c_int), P(C.c_double)]
        _LIB = L
    return _LIB


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


def apply_gate(sub: np.ndarray, positions, matrix: np.ndarray) -> None:
    """In place on sub (p, 2^nl) complex128; positions[j] <-> matrix bit j."""
    p, per = sub.shape
    nl = per.bit_length() - 1
    pos, pp = _iptr(positions)
    u = np.ascontiguousarray(matrix, dtype=np.complex128)
    lib().orc_apply_gate(_dptr(sub), p, nl, len(pos), pp, _dptr(u))


def perform_qr(sub: np.ndarray, dest) -> int:
    p, per = sub.shape
    nl = per.bit_length() - 1
    n = nl + (p.bit_length() - 1)
    scratch = np.empty_like(sub)
    d, dp = _iptr(dest)
    return int(lib().orc_perform_qr(_dptr(sub), _dptr(scratch), p, nl, n, dp))


def mask_term(letters: str, pos_of, n_local: int) -> MaskedTerm:
    m = MaskedTerm()
    po, pp = _iptr(pos_of)
    if lib().orc_mask_term(letters.encode(), len(letters), pp, n_local, C.byref(m)) != 0:
        raise ValueError("NotDiagonalizable: global X/Y letter")
    return m


def expectation_tile(sub: np.ndarray, masked: list[MaskedTerm], coeffs) -> np.ndarray:
    """partial[pe] for one plan tile (dist_sim.cpp:289-295)."""
    p, per = sub.shape
    nl = per.bit_length() - 1
    arr = (MaskedTerm * max(1, len(masked)))(*masked)
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.complex128))
    partial = np.zeros(p, dtype=np.complex128)
    lib().orc_expectation_tile(_dptr(sub), p, nl, len(masked), arr, _dptr(c), _dptr(partial))
    return partial


def flatten(sub: np.ndarray, qubit_at) -> np.ndarray:
    p, per = sub.shape
    nl = per.bit_length() - 1
    n = nl + (p.bit_length() - 1)
    out = np.empty(p * per, dtype=np.complex128)
    q, qp = _iptr(qubit_at)
    lib().orc_flatten(_dptr(sub), p, nl, n, qp, _dptr(out))
    return out


class Layout:
    """Logical layout bookkeeping for the oracle (layout.cpp:25-40, 96-112)."""

    def __init__(self, n: int, p: int):
        self.n, self.nl = n, n - (p.bit_length() - 1)
        self.pos_of = list(range(n))
        self.qubit_at = list(range(n))

    def dest_for(self, after_pos_of) -> list[int]:
        # dest[p] = after.pos_of[before.qubit_at[p]] (dist_sim.cpp:213-219)
        return [after_pos_of[self.qubit_at[p]] for p in range(self.n)]

    def adopt(self, after_pos_of) -> None:
        self.pos_of = list(after_pos_of)
        for q, p in enumerate(self.pos_of):
            self.qubit_at[p] = q


def run_qsu(n: int, p: int, circuit, schedule) -> tuple[np.ndarray, Layout, list[int]]:
    """Reference run_qsu (dist_sim.cpp:242-252) from |0>, driven by a product
    Schedule object (its event layouts are checked bit-exact separately)."""
    sub = np.zeros((p, 1 << (n - (p.bit_length() - 1))), dtype=np.complex128)
    sub[0, 0] = 1.0
    lay = Layout(n, p)
    moved = []
    ev_i = 0
    events = schedule.qr_events
    for t, tile in enumerate(schedule.tiles):
        while ev_i < len(events) and events[ev_i].before_tile == t:
            ev = events[ev_i]
            moved.append(perform_qr(sub, lay.dest_for(ev.after.pos_of)))
            lay.adopt(ev.after.pos_of)
            ev_i += 1
        for gid in tile.gates:
            op = circuit.operators[gid]
            apply_gate(sub, [lay.pos_of[q] for q in op.targets], op.payload)
    return sub, lay, moved
