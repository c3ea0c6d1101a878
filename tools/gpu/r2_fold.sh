#!/bin/bash
# Same-box A/B: PE sign mask folded into the group mf (product) vs libqrt_nofold.so
O=${OUT:-gpurun_out/fold}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_abi.py -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
P=$PWD/paper_2410_04252_b200
for i in 1 2; do
  for v in base nofold; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni30_${v}_$i.json 2>&1
  done
done
