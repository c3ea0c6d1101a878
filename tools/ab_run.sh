# scratch: single-bit EVC bodies split by table mode
O=gpurun_out/ab19; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evc.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea --hamiltonian uniform --terms 1000 > $O/uni.json 2>&1
python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea > $O/hea.json 2>&1
