#!/bin/bash
# ncu launch list of one default bench step (C3 32q) on the final tree (serialised, cold-cache per launch)
O=${OUT:-gpurun_out/launch5}; mkdir -p $O
timeout 1500 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $O/launches_32q.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo rc=$? >> $O/ncu_launch.log
