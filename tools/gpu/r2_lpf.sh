#!/bin/bash
# Same-box A/B: light passes with the next op's dispatch code prefetched (product) vs libqrt_nolpf.so
O=${OUT:-gpurun_out/lpf}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_light.py tests/test_gpu_parity.py -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
P=$PWD/paper_2410_04252_b200
for i in 1 2; do
  for v in base nolpf; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
  done
done
