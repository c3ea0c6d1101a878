#!/bin/bash
# EVC per-set overheads: same-box A/B of the host set tables (QRT_EVC_SET_TABLES=1/0); the
# present-mask guard is in both arms
O=${OUT:-gpurun_out/r2evcfill}; mkdir -p $O
for i in 1 2; do
  for t in 1 0; do
    QRT_EVC_FILL=$t timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_t${t}_$i.json 2>&1
    QRT_EVC_FILL=$t timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni4000_t${t}_$i.json 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_checked.py -q -x --timeout 300 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
