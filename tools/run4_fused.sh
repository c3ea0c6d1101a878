timeout 400 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi4.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi4.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for f in 1 0; do QRT_FUSED_QR=$f timeout 300 $R --master-port 2955$f bench.py --gpus 4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/b30_n4_f$f.json 2> gpurun_out/b30_n4_f$f.err; done
timeout 500 $R --master-port 29561 bench.py --gpus 4 --qubits 34 --circuit hea --steps 1 --warmup 1 > gpurun_out/b34h_n4.json 2> gpurun_out/b34h_n4.err
timeout 500 $R --master-port 29562 bench.py --gpus 4 --qubits 32 --steps 1 --warmup 1 > gpurun_out/b32_n4.json 2> gpurun_out/b32_n4.err
