#!/bin/bash
# Same-box A/B of EVC compile-time variants on the JW passes (30q HEA): product vs early0 / acc2 / acc8
O=${OUT:-gpurun_out/evcvar}; mkdir -p $O
P=$PWD/paper_2410_04252_b200
for i in 1 2; do
  for v in base early0 acc2 acc8; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
  done
done
