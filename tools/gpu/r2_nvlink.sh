#!/bin/bash
# N-GPU NVLink QR evidence (single process): event-timed rates, then ncu NVLink counters.
O=${OUT:-gpurun_out/r2nvl$(nvidia-smi -L | wc -l)}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > $O/topo.txt 2>&1
[ -x tools/mb_imma ] && timeout 120 tools/mb_imma > $O/mb_imma.txt 2>&1
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
if [ "$N" = "2" ]; then
  # 34 qubits on 2 GPUs: 128 GiB per GPU, so the QR must run in place (auto)
  BENCH_DEBUG=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus 2 --qubits 34 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench34_gf_n2.json 2> $O/bench34_gf_n2.err
fi
if [ "$N" = "4" ]; then
  for circ in gatefabric hea; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 \
       bench.py --gpus 4 --qubits 30 --circuit $circ --steps 2 --warmup 3 --no-cpu-baseline > $O/bench30_${circ}_n4.json 2> $O/bench30_${circ}_n4.err
  done
  for circ in hea; do
    BENCH_DEBUG=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
       bench.py --gpus 4 --qubits 34 --circuit $circ --steps 2 --warmup 3 --no-cpu-baseline > $O/bench34_${circ}_n4.json 2> $O/bench34_${circ}_n4.err
  done
  BENCH_DEBUG=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 \
     bench.py --gpus 4 --qubits 34 --circuit hea --hamiltonian uniform --terms 10000 --steps 1 --warmup 3 --no-cpu-baseline > $O/bench34_c5_n4.json 2> $O/bench34_c5_n4.err
fi
