#!/bin/bash
# N-GPU NVLink QR evidence (single process): event-timed rates, then ncu NVLink counters.
O=${OUT:-gpurun_out/r2nvl}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 600 python tools/qr_nvlink.py --nl 30 --iters 5 > $O/qr_nl30_n$N.jsonl 2> $O/qr.err
timeout 600 python tools/qr_nvlink.py --nl 31 --iters 3 > $O/qr_nl31_n$N.jsonl 2>> $O/qr.err
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --csv --log-file $O/ncu_qr_n$N.csv python tools/qr_nvlink.py --nl 28 --iters 1 > $O/ncu_qr.log 2>&1
# multi-process: distributed parity tests + 32q C3 step at N with push vs in-place QR
timeout 900 python -m pytest tests/test_gpu_multi.py -q > $O/multi.log 2>&1; echo rc=$? >> $O/multi.log
for ip in 0 1; do
  QRT_QR_INPLACE=$ip BENCH_DEBUG=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $N --steps 2 --warmup 3 --no-cpu-baseline > $O/bench32_n${N}_inplace$ip.json 2> $O/bench32_n${N}_inplace$ip.err
done
