#!/bin/bash
O=gpurun_out/r2dbg; mkdir -p $O
for args in "18 500 1,2,4,8" "18 2000 1,2,4,8" "20 2000 1,2,4,8" "16 2000 1,2,4,8"; do
  timeout 300 python tools/dbg_uniform.py $args >> $O/base.txt 2>&1
done
for knob in QRT_EVC_LINEAR=0 QRT_EVC_PIPE=0 QRT_EVC_COSET=0 QRT_PLAN_CACHE=0 QRT_EVC_GLOBAL_COVER=0; do
  echo "$knob" >> $O/knobs.txt
  env $knob timeout 300 python tools/dbg_uniform.py 18 2000 1,2,8 >> $O/knobs.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_inplace.py tests/test_gpu_multi.py -q -x > $O/inplace.log 2>&1; echo rc=$? >> $O/inplace.log
