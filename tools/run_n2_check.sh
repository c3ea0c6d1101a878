#!/bin/bash
# Two-GPU check (gpurun --gpus 2): multi-process GPU tests and the default
# bench at N = 2, twice with per-step times (the intermittent EVC stall).
OUT=${OUT:-gpurun_out/n2}
mkdir -p "$OUT"
R() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2" "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > "$OUT/tests_multi.log" 2>&1; echo "rc=$?" >> "$OUT/tests_multi.log"
for i in 1 2; do
BENCH_DEBUG=1 R 2 2955$i bench.py --gpus 2 --steps 4 --warmup 3 > "$OUT/b30_gf_n2_$i.json" 2> "$OUT/b30_gf_n2_$i.err"
done
echo done > "$OUT/done"
