#!/bin/bash
# EVC single-bit-group path for GF(2)-linear passes (QRT_EVC_SINGLE): tests, then same-box A/B
O=${OUT:-gpurun_out/single2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_abi.py -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for rep in 1 2; do
  for v in 0 1; do
    QRT_EVC_SINGLE=$v timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --steps 3 --warmup 3 --no-cpu-baseline > $O/uni30_s${v}_$rep.json 2> $O/uni30_s${v}_$rep.err
    QRT_EVC_SINGLE=$v timeout 600 python bench.py --qubits 30 --circuit hea --steps 3 --warmup 3 --no-cpu-baseline > $O/hea30_s${v}_$rep.json 2> $O/hea30_s${v}_$rep.err
  done
done
