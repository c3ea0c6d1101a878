#!/bin/bash
# EVC per-set tables precomputed on the host: same-box A/B (QRT_EVC_SET_TABLES=1/0, interleaved)
O=${OUT:-gpurun_out/r2evcset2}; mkdir -p $O
for i in 1 2; do
  for t in 1 0; do
    QRT_EVC_SET_TABLES=$t timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_t${t}_$i.json 2>&1
    QRT_EVC_SET_TABLES=$t timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni4000_t${t}_$i.json 2>&1
  done
done
