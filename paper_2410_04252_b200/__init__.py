"""B200-native QSU / QR / EVC hot path of arXiv 2410.04252 (lazy qubit reordering).

The package is a thin Python face over native code:

* ``libqrt.so`` — hand-written sm_100a CUDA kernels behind the C ABI of
  ``include/qrt.h`` (gate passes, NVLink reorder, batched Pauli expectation);
* ``libqrtile_b200.so`` — the reference's C++ ``qrtile`` API re-implemented
  host-side (schedulers bit-exact with the reference) on top of libqrt;
* ``_qrtile`` — pybind11 bindings of that API.

There is no CPU fallback: importing the package without the native libraries,
or running on a machine without an sm_100 GPU, fails loudly at the first
device call (``DeviceError``).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent

try:
    from . import _qrtile  # noqa: F401  (loads libqrtile_b200.so and libqrt.so)
except ImportError as exc:  # pragma: no cover - explicit, loud failure
    raise ImportError(
        "paper_2410_04252_b200 native extension is not built; run "
        "`python -m paper_2410_04252_b200.build` (needs nvcc for sm_100a)") from exc

from ._qrtile import *  # noqa: F401,F403,E402
from ._qrtile import Error, DeviceError  # noqa: E402


def libqrt_path() -> str:
    return str(_PKG / "libqrt.so")


def load_libqrt() -> ctypes.CDLL:
    """The C ABI library itself (for direct ctypes callers and ABI tests)."""
    return ctypes.CDLL(libqrt_path())


def inplace_reorder_plan(n: int, p: int, dest) -> tuple[list, list, list]:
    """The in-place decomposition libqrt uses for qrt_reorder(dest) on a
    single-buffer state (qrt_reorder_inplace_plan): two passes of disjoint
    local position transpositions, then the (local slot, PE bit) pairs that
    are swapped between PEs.  Host only."""
    lib = load_libqrt()
    a0, a1, cr = (ctypes.c_int * 128)(), (ctypes.c_int * 128)(), (ctypes.c_int * 128)()
    n0, n1, k = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = lib.qrt_reorder_inplace_plan(n, p, (ctypes.c_int * n)(*dest), a0, ctypes.byref(n0), a1, ctypes.byref(n1),
                                      cr, ctypes.byref(k))
    if rc != 0:
        lib.qrt_last_error.restype = ctypes.c_char_p
        raise Error(lib.qrt_last_error().decode())
    pairs = lambda arr, c: [(arr[2 * i], arr[2 * i + 1]) for i in range(c.value)]  # noqa: E731
    return pairs(a0, n0), pairs(a1, n1), pairs(cr, k)


def state_mode(state) -> dict:
    """QR mode of a live state: {"inplace_qr": bool, "sm_count": int}."""
    lib = load_libqrt()
    ip, sm = ctypes.c_int(), ctypes.c_int()
    rc = lib.qrt_state_mode(ctypes.c_void_p(state.handle()), ctypes.byref(ip), ctypes.byref(sm))
    if rc != 0:
        raise Error("qrt_state_mode failed")
    return {"inplace_qr": bool(ip.value), "sm_count": sm.value}


def init_distributed(device: int | None = None):
    """One process per GPU: read RANK/WORLD_SIZE/LOCAL_RANK, share the NCCL id
    over torch.distributed (gloo, plumbing only) and create the libqrt
    communicator.  Returns (rank, world, device)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    dev = local if device is None else device
    if world == 1:
        _qrtile.init_device(0, 1, dev)
        return 0, 1, dev
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("gloo")
    box = [_qrtile.device_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    _qrtile.init_device(rank, world, dev, box[0])
    return rank, world, dev
