"""The checked build (libqrt_checked.so, -DQRT_CHECKS): device-side bounds
checks in every exchange / gate / EVC kernel and, in the pipelined EVC
kernels, a check that the awaited buffer really holds the awaited tile (the
property the round-1 mbarrier race violated).  compute-sanitizer is closed on
the GPU pool; this is the substitute: tests/checked_worker.py runs small cases
of every kernel family against the oracle with the checked library preloaded."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_checked_build_small_cases():
    lib = ROOT / "paper_2410_04252_b200" / "libqrt_checked.so"
    assert lib.exists(), "build() did not produce libqrt_checked.so"
    env = dict(os.environ, LD_PRELOAD=str(lib))
    res = subprocess.run([sys.executable, str(ROOT / "tests" / "checked_worker.py")], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert res.stdout.strip().startswith("ok")
