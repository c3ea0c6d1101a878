#!/bin/bash
# EVC per-set tables precomputed on the host (A/B vs 918-950 ms of earlier runs); EVC tests
O=${OUT:-gpurun_out/r2evcset}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_abi.py tests/test_gpu_checked.py -q -x --timeout 300 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for i in 1 2; do
  timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_$i.json 2>&1
done
timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni4000.json 2>&1
