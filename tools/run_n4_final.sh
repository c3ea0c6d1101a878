#!/bin/bash
# Four-GPU round-end measurements (gpurun --gpus 4): multi-process tests, the
# default bench and HEA at N = 4, then the C5 stress (uniform 10k words at 32/34q).
OUT=${OUT:-gpurun_out/n4}
mkdir -p "$OUT"
R() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2" "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > "$OUT/tests_multi.log" 2>&1; echo "rc=$?" >> "$OUT/tests_multi.log"
BENCH_DEBUG=1 R 4 29561 bench.py --gpus 4 --steps 4 --warmup 3 > "$OUT/b30_gf_n4.json" 2> "$OUT/b30_gf_n4.err"
BENCH_DEBUG=1 R 4 29562 bench.py --gpus 4 --circuit hea --steps 4 --warmup 3 > "$OUT/b30_hea_n4.json" 2> "$OUT/b30_hea_n4.err"
OUT=$OUT/c5 bash tools/run_c5.sh
echo done > "$OUT/done"
