#!/bin/bash
# Round profiling on the GPU box (run from the repo root under gpurun):
# bench lines, the kernel launch list of the default bench, and one
# `ncu --set full` capture of each top kernel.  Each ncu command runs only
# after the same command exited 0 without ncu (the bench lines above).
OUT=${OUT:-gpurun_out/prof}
mkdir -p "$OUT"
NCU="ncu --clock-control none"
python bench.py > "$OUT/bench30_gf.json" 2> "$OUT/bench30_gf.err" || exit 1
python bench.py --circuit hea > "$OUT/bench30_hea.json" 2> "$OUT/bench30_hea.err" || exit 1
$NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/launches_30q_gf.csv" \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_launch_gf.log" 2>&1
$NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/launches_30q_hea.csv" \
    python bench.py --circuit hea --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_launch_hea.log" 2>&1
$NCU --set full --import-source on -k regex:gate_pass -s 10 -c 1 -o "$OUT/gate30" \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_gate.log" 2>&1
$NCU --set full --import-source on -k regex:coset_pipe -s 10 -c 1 -o "$OUT/coset30" \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_coset.log" 2>&1
$NCU --set full --import-source on -k regex:light_pass -s 10 -c 1 -o "$OUT/light30" \
    python bench.py --circuit hea --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_light.log" 2>&1
echo done
