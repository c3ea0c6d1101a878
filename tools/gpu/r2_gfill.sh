#!/bin/bash
# Gate-pass tile load/store with the linear swizzle (A/B vs the previous build's 30q / 32q lines)
O=${OUT:-gpurun_out/r2gfill}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_light.py -q -x --timeout 300 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30.json 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 > $O/gf32.json 2>&1
