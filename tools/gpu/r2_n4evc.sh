#!/bin/bash
# 4-GPU lines of the EVC-heavy configs after the EVC latency work: C5 stress (34q, 10k words), C4 HEA 34q, C3 32q
O=${OUT:-gpurun_out/n4evc}; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555"
timeout 1200 $R bench.py --gpus 4 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench34_c5_n4.json 2> $O/bench34_c5_n4.err
timeout 900 $R bench.py --gpus 4 --qubits 34 --circuit hea --steps 3 --warmup 3 --no-cpu-baseline > $O/bench34_hea_n4.json 2> $O/bench34_hea_n4.err
timeout 900 $R bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench32_n4.json 2> $O/bench32_n4.err
