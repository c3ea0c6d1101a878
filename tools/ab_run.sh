# scratch A/B script for gpurun (edited per experiment)
O=gpurun_out/ab16; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evc.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for pp in 1 0; do
QRT_EVC_PIPE=$pp python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea > $O/hea_jw_$pp.json 2>&1
QRT_EVC_PIPE=$pp python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea --hamiltonian uniform --terms 1000 > $O/uni_$pp.json 2>&1
done
