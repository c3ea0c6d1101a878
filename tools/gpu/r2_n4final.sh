#!/bin/bash
# Final tree on 4 GPUs: multi-process tests, C3 32q at N = 2 / 4, C4 HEA 34q and C5 34q at N = 4
O=${OUT:-gpurun_out/n4final}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/multi.log 2>&1; echo rc=$? >> $O/multi.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561"
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562"
timeout 900 $R2 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench32_n2.json 2> $O/bench32_n2.err
timeout 900 $R4 bench.py --gpus 4 --steps 3 --warmup 3 > $O/bench32_n4.json 2> $O/bench32_n4.err
timeout 900 $R4 bench.py --gpus 4 --qubits 34 --circuit hea --steps 3 --warmup 3 --no-cpu-baseline > $O/bench34_hea_n4.json 2> $O/bench34_hea_n4.err
timeout 1200 $R4 bench.py --gpus 4 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench34_c5_n4.json 2> $O/bench34_c5_n4.err
