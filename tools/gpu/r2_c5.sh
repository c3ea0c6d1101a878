#!/bin/bash
# C5 (10,000 reference-Rng words at 34q after the HEA QSU) on 4 GPUs at p = 4 and p = 8 after the
# per-set EVC overhead fixes; C4 at p = 4 for the record
O=${OUT:-gpurun_out/r2c5}; mkdir -p $O
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 4 "${@:3}"; }
BENCH_DEBUG=1 run 1800 29571 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_c5_p4.json 2> $O/bench34_c5_p4.err
BENCH_DEBUG=1 run 1800 29572 --pes-per-gpu 2 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_c5_p8.json 2> $O/bench34_c5_p8.err
BENCH_DEBUG=1 run 1200 29573 --qubits 34 --circuit hea --no-cpu-baseline > $O/bench34_hea_p4.json 2> $O/bench34_hea_p4.err
