#!/bin/bash
# BASELINE C5 stress on one box (gpurun --gpus 4): EVC of 10,000 uniformly random
# Pauli words after a HEA QSU at 32 and 34 qubits (GF(2)-linear, pipelined coset passes).
OUT=${OUT:-gpurun_out/c5c}
mkdir -p "$OUT"
R() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2" "${@:3}"; }
BENCH_DEBUG=1 R 4 29532 bench.py --gpus 4 --qubits 32 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 \
    > "$OUT/b32_uni10k_n4.json" 2> "$OUT/b32_uni10k_n4.err"
BENCH_DEBUG=1 R 4 29531 bench.py --gpus 4 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 \
    > "$OUT/b34_uni10k_n4.json" 2> "$OUT/b34_uni10k_n4.err"
echo done > "$OUT/done"
