#!/bin/bash
# Strong-scaling record of the default bench (C3, 32q) at N = nvidia-smi GPUs with the final
# build, plus the multi-process tests; at N = 2 also 34q (single buffer), at N = 4 also p = 8.
O=${OUT:-gpurun_out/r2scale$(nvidia-smi -L | wc -l)}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $N "${@:3}"; }
BENCH_DEBUG=1 run 1200 29561 > $O/bench32_n$N.json 2> $O/bench32_n$N.err
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $O/multi.log 2>&1; echo rc=$? >> $O/multi.log
if [ "$N" = "2" ]; then
  BENCH_DEBUG=1 run 1800 29562 --qubits 34 --no-cpu-baseline > $O/bench34_n2.json 2> $O/bench34_n2.err
fi
if [ "$N" = "4" ]; then
  BENCH_DEBUG=1 run 1200 29563 --pes-per-gpu 2 --no-cpu-baseline > $O/bench32_p8_n4.json 2> $O/bench32_p8_n4.err
fi
