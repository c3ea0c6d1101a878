#!/bin/bash
O=${OUT:-gpurun_out/r2teams}; mkdir -p $O
for t in 2 1 0; do
  QRT_EVC_TEAMS=$t timeout 900 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni4000_t$t.json 2>&1
  QRT_EVC_TEAMS=$t timeout 900 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 2 --warmup 3 > $O/jw_t$t.json 2>&1
done
QRT_EVC_TEAMS=1 timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py -q -x --timeout 300 -k "uniform or coset or linear" > $O/tests_t1.log 2>&1; echo rc=$? >> $O/tests_t1.log
