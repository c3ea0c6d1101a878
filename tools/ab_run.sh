# scratch: light pass in-place register updates
O=gpurun_out/ab18; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_light.py tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea > $O/hea.json 2>&1
