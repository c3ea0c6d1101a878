#!/bin/bash
# Final strong-scaling lines (gpurun --gpus 4): default bench and HEA at N = 2, 4; 34q HEA at N = 4.
OUT=${OUT:-gpurun_out/scale_short}
mkdir -p "$OUT"
R() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2" "${@:3}"; }
BENCH_DEBUG=1 R 2 29711 bench.py --gpus 2 > "$OUT/b30_gf_n2.json" 2> "$OUT/b30_gf_n2.err"
BENCH_DEBUG=1 R 4 29712 bench.py --gpus 4 > "$OUT/b30_gf_n4.json" 2> "$OUT/b30_gf_n4.err"
BENCH_DEBUG=1 R 2 29713 bench.py --gpus 2 --circuit hea > "$OUT/b30_hea_n2.json" 2> "$OUT/b30_hea_n2.err"
BENCH_DEBUG=1 R 4 29714 bench.py --gpus 4 --circuit hea > "$OUT/b30_hea_n4.json" 2> "$OUT/b30_hea_n4.err"
BENCH_DEBUG=1 R 4 29715 bench.py --gpus 4 --qubits 34 --circuit hea --steps 2 --warmup 3 > "$OUT/b34_hea_n4.json" 2> "$OUT/b34_hea_n4.err"
echo done > "$OUT/done"
