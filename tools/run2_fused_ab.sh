timeout 300 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi2.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi2.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for f in 1 0; do QRT_FUSED_QR=$f timeout 300 $R --master-port 2953$f bench.py --gpus 2 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/b30_n2_f$f.json 2> gpurun_out/b30_n2_f$f.err; done
for f in 1 0; do QRT_FUSED_QR=$f timeout 300 $R --master-port 2954$f bench.py --gpus 2 --circuit hea --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/b30h_n2_f$f.json 2> gpurun_out/b30h_n2_f$f.err; done
