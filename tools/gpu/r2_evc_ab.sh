#!/bin/bash
# EVC fill A/B (QRT_EVC_FILL) on 30q GateFabric + JW, then compute-sanitizer on the small cases
O=${OUT:-gpurun_out/r2ab}; mkdir -p $O
for f in 1 0; do
  QRT_EVC_FILL=$f timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_fill$f.json 2>&1
done
QRT_EVC_FILL=1 timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_fill1b.json 2>&1
