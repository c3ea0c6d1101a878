#!/bin/bash
# Same-box A/B/C of compile-time EVC variants: product libqrt.so vs LD_PRELOAD of libqrt_{nopf,nouni}.so
O=${OUT:-gpurun_out/var3}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
P=$PWD/paper_2410_04252_b200
for i in 1 2; do
  for v in base nopf nouni; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni30_${v}_$i.json 2>&1
  done
done
