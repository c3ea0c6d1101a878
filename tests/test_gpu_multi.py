"""Multi-GPU path (one process per GPU): QR over NVLink peer stores, NCCL
partial gathers.  Runs tests/mp_worker.py under torch.distributed.run on 2
(and 4 when present) GPUs of the box; skipped on a single-GPU box."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_qsu_evc(qb, world):
    if qb.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), str(ROOT / "tests" / "mp_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ))
    assert res.returncode == 0, res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["ok"], out


def test_qr_bench_single_process(qb):
    """qrt_qr_bench (tools/qr_nvlink.py): both exchange kernels over CUDA peer
    access in one process, k = 1..log2(N); rates are positive and finite."""
    import ctypes as C

    n = qb.device_count()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    n = 4 if n >= 4 else 2
    lib = qb.load_libqrt()
    for inplace in (0, 1):
        for k in range(1, n.bit_length()):
            ms, gbs = C.c_double(), C.c_double()
            assert lib.qrt_qr_bench(n, 24, k, inplace, 2, C.byref(ms), C.byref(gbs)) == 0
            assert ms.value > 0 and 0 < gbs.value < 5000
