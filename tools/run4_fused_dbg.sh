R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
mkdir -p gpurun_out/trace4
BENCH_DEBUG=1 QRT_TRACE=gpurun_out/trace4/t timeout 300 $R --master-port 29571 bench.py --gpus 4 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b30_n4_dbg.json 2> gpurun_out/b30_n4_dbg.err
BENCH_DEBUG=1 QRT_FUSED_QR=0 timeout 300 $R --master-port 29572 bench.py --gpus 4 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/b30_n4_dbg0.json 2> gpurun_out/b30_n4_dbg0.err
