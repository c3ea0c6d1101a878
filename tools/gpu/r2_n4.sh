#!/bin/bash
# 4-GPU re-check after the XOR exchange schedule: microbench, multi tests, in-place steps at 32/34q
O=${OUT:-gpurun_out/r2n4b}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
timeout 600 python tools/qr_nvlink.py --nl 30 --iters 5 > $O/qr_nl30_n$N.jsonl 2> $O/qr.err
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --csv --log-file $O/ncu_qr_n$N.csv python tools/qr_nvlink.py --nl 28 --iters 1 > $O/ncu_qr.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $O/multi.log 2>&1; echo rc=$? >> $O/multi.log
QRT_QR_INPLACE=1 BENCH_DEBUG=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus $N --steps 2 --warmup 3 --no-cpu-baseline > $O/bench32_n${N}_inplace1.json 2> $O/bench32_n${N}_inplace1.err
BENCH_DEBUG=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
   bench.py --gpus 4 --qubits 34 --circuit hea --steps 2 --warmup 3 --no-cpu-baseline > $O/bench34_hea_n4.json 2> $O/bench34_hea_n4.err
BENCH_DEBUG=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 \
   bench.py --gpus 4 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_c5_n4.json 2> $O/bench34_c5_n4.err
