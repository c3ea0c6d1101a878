#!/bin/bash
O=gpurun_out/r2dbg2; mkdir -p $O
timeout 600 python tools/dbg_uniform.py 24 2000 1,2,4,8 >> $O/base.txt 2>&1
for args in "22 2000 1,2,4,8" "23 2000 1,2,4,8" "21 2000 1,2,4,8" "24 500 1,2,4,8" ; do
  timeout 300 python tools/dbg_uniform.py $args nooracle >> $O/base.txt 2>&1
done
for knob in QRT_EVC_LINEAR=0 QRT_EVC_PIPE=0 QRT_EVC_COSET=0 QRT_EVC_GLOBAL_COVER=0 QRT_DEBUG_PLAN=1; do
  echo "$knob" >> $O/knobs.txt
  env $knob timeout 300 python tools/dbg_uniform.py 24 2000 1,2,8 nooracle >> $O/knobs.txt 2>&1
done
