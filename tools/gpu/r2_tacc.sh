#!/bin/bash
# Same-box A/B: per-thread accumulation with table sign flips (libqrt_tacc.so) vs the product; parity under the variant
O=${OUT:-gpurun_out/tacc}; mkdir -p $O
P=$PWD/paper_2410_04252_b200
LD_PRELOAD=$P/libqrt_tacc.so timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py -q -m gpu > $O/tests_tacc.log 2>&1; echo rc=$? >> $O/tests_tacc.log
for i in 1 2; do
  for v in base tacc; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_${v}_$i.json 2>&1
  done
done
