"""bench.py's JSON contract, on a small workload: the reference arm on CPU
(the unmodified reference from oracle/_ref, never the product) and our arm on
the GPU.  Keys per the driver contract: metric/value/unit, steps/warmup,
higher_is_better, e2e with H2D/D2H bytes, roofline, cpu_baseline, clocks,
gpu_launches, config.workload."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _line(args, timeout=300):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert res.returncode == 0, res.stderr[-2000:]
    return json.loads([l for l in res.stdout.splitlines() if l.startswith("{")][-1])


def test_reference_arm_contract(ref):
    d = _line(["--impl", "reference", "--qubits", "16", "--cpu-sample-qubits", "12", "--cpu-full-qubits", "12", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["nproc"] >= 1 and "sample" in cb
    assert cb["counts"]["n_gates"] == 16 * 4 * 7  # gatefabric_block_count(16, 64) = 64 * (4 + 3)
    # the reference arm never maps the product's libraries
    assert all("_ref" in so or "oracle" in so for so in d["native_so_loaded"]), d["native_so_loaded"]
    assert d["config"]["qubits"] == 16 and "workload" in d["config"]
    assert "extrapolated" in cb["sample"]  # 16 > --cpu-full-qubits 12: bounded sample


def test_reference_arm_full_run(ref):
    """Small workloads (n <= --cpu-full-qubits) run the reference's whole
    evaluate_energy: measured, not extrapolated."""
    d = _line(["--impl", "reference", "--qubits", "12", "--cpu-full-qubits", "12", "--pes-per-gpu", "4",
               "--steps", "1", "--warmup", "0"])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and "measured" in cb["sample"] and d["value"] > 0
    assert d["config"]["pes"] == 4


@pytest.mark.gpu
def test_ours_arm_contract():
    d = _line(["--qubits", "16", "--steps", "1", "--warmup", "1", "--cpu-sample-qubits", "12"], timeout=600)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["roofline"]["bound"] in ("hbm", "tensor") and d["roofline"]["peak"] > 0
    assert any("libqrt.so" in so for so in d["native_so_loaded"])
    assert d["cpu_baseline"]["kind"] == "reference"
