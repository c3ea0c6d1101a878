#!/bin/bash
# C4 (HEA 34q) at p = 8 on 4 GPUs after the light-pass fusion limit, and the default C3 line at N = 4
O=${OUT:-gpurun_out/r2c4}; mkdir -p $O
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 4 "${@:3}"; }
BENCH_DEBUG=1 run 1200 29551 --pes-per-gpu 2 --qubits 34 --circuit hea --no-cpu-baseline > $O/bench34_hea_p8_n4.json 2> $O/bench34_hea_p8_n4.err
BENCH_DEBUG=1 run 1200 29552 > $O/bench32_n4.json 2> $O/bench32_n4.err
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $O/multi.log 2>&1; echo rc=$? >> $O/multi.log
