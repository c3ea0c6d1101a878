mkdir -p gpurun_out/ab1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evc.py -x -q > gpurun_out/ab1/tests.log 2>&1; echo rc=$? >> gpurun_out/ab1/tests.log
QRT_GAUSS=0 python bench.py --no-cpu-baseline > gpurun_out/ab1/real.json 2>&1
python bench.py --no-cpu-baseline > gpurun_out/ab1/gauss.json 2>&1
