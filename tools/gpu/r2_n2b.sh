#!/bin/bash
# 2-GPU follow-ups: the default C3 line at N=2 (with cpu_baseline), the fused pull QR at 2^31
# amplitudes per PE (the 34q/p=8 regime) vs in place, and 34q eager (adhoc) with in-place QRs.
O=${OUT:-gpurun_out/r2n2b}; mkdir -p $O
run() { timeout $1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus 2 "${@:3}"; }
BENCH_DEBUG=1 run 900 29521 > $O/bench32_n2.json 2> $O/bench32_n2.err
QRT_QR_INPLACE=0 QRT_FUSED_QR_MAX_LOG2=31 BENCH_DEBUG=1 run 900 29522 --no-cpu-baseline > $O/bench32_n2_fused31.json 2> $O/bench32_n2_fused31.err
BENCH_DEBUG=1 run 2400 29523 --qubits 34 --schedule adhoc --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_adhoc_n2.json 2> $O/bench34_adhoc_n2.err
