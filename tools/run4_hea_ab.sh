R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for f in 1 0; do BENCH_DEBUG=1 QRT_FUSED_QR=$f timeout 300 $R --master-port 2959$f bench.py --gpus 4 --circuit hea --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/h30_n4_$f.json 2> gpurun_out/h30_n4_$f.err; done
for f in 1 0; do BENCH_DEBUG=1 QRT_FUSED_QR=$f timeout 600 $R --master-port 2960$f bench.py --gpus 4 --qubits 34 --circuit hea --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/h34_n4_$f.json 2> gpurun_out/h34_n4_$f.err; done
