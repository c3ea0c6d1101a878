#!/bin/bash
# Lazy vs eager at the metric's configuration on 4 GPUs (p = 4, and p = 8 with 2 PEs per GPU)
O=${OUT:-gpurun_out/r2eager}; mkdir -p $O
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 4 "${@:3}"; }
BENCH_DEBUG=1 run 1200 29541 --schedule adhoc --no-cpu-baseline > $O/bench32_adhoc_p4.json 2> $O/bench32_adhoc_p4.err
BENCH_DEBUG=1 run 1200 29542 --pes-per-gpu 2 --schedule adhoc --no-cpu-baseline > $O/bench32_adhoc_p8.json 2> $O/bench32_adhoc_p8.err
BENCH_DEBUG=1 run 1800 29543 --pes-per-gpu 2 --qubits 34 --circuit hea --schedule adhoc --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_hea_adhoc_p8.json 2> $O/bench34_hea_adhoc_p8.err
