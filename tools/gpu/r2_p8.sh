#!/bin/bash
# The p = 8 configurations (BASELINE C3 at p=8, C4, C5) on 4 GPUs with 2 PEs per GPU:
# the reference's p = 8 schedules and plans (k = 3 QRs, 8-way exchanges) on hardware.
O=${OUT:-gpurun_out/r2p8}; mkdir -p $O
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 4 --pes-per-gpu 2 "${@:3}"; }
BENCH_DEBUG=1 run 900 29531 --no-cpu-baseline > $O/bench32_p8_n4.json 2> $O/bench32_p8_n4.err
BENCH_DEBUG=1 run 1200 29532 --qubits 34 --circuit hea --no-cpu-baseline > $O/bench34_hea_p8_n4.json 2> $O/bench34_hea_p8_n4.err
BENCH_DEBUG=1 run 2400 29533 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_c5_p8_n4.json 2> $O/bench34_c5_p8_n4.err
timeout 600 python tools/qr_nvlink.py --nl 30 --iters 5 > $O/qr_nl30_n4.jsonl 2> $O/qr.err
