#!/bin/bash
# Linear-pass coalescing A/B (QRT_EVC_LINEAR_COAL = unit low positions of a GF(2) tile):
# 30q HEA + 1,000 / 4,000 uniform words (reference Rng(2024)), 1 GPU
O=${OUT:-gpurun_out/r2lin}; mkdir -p $O
for c in ${COALS:-0 1 2}; do
  for t in 1000 4000; do
    QRT_EVC_LINEAR_COAL=$c timeout 900 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms $t \
       --no-cpu-baseline --steps 2 --warmup 3 > $O/hea30_uni${t}_coal$c.json 2>&1
  done
done
QRT_EVC_LINEAR_COAL=0 timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x --timeout 300 -k "uniform or linear" > $O/tests_coal0.log 2>&1; echo rc=$? >> $O/tests_coal0.log
