# scratch A/B script for gpurun (edited per experiment)
O=gpurun_out/ab14; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evc.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea --hamiltonian uniform --terms 1000 > $O/uni_lin.json 2>&1
QRT_EVC_LINEAR=0 python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea --hamiltonian uniform --terms 1000 > $O/uni_wide.json 2>&1
python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea > $O/hea_jw.json 2>&1
