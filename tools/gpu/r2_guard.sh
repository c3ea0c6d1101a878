#!/bin/bash
# Same-box A/B of the EVC set-overhead changes on Jordan-Wigner passes (30q and 32q GateFabric)
O=${OUT:-gpurun_out/r2guard}; mkdir -p $O
for i in 1 2; do
  for cfg in "1 1" "0 1" "1 0" "0 0"; do
    set -- $cfg
    QRT_EVC_PRESENT_GUARD=$1 QRT_EVC_SET_TABLES=$2 timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_g$1_t$2_$i.json 2>&1
  done
done
for cfg in "1 1" "0 0"; do
  set -- $cfg
  QRT_EVC_PRESENT_GUARD=$1 QRT_EVC_SET_TABLES=$2 timeout 900 python bench.py --no-cpu-baseline --steps 2 --warmup 3 > $O/gf32_g$1_t$2.json 2>&1
done
