# scratch: linear-tile coalescing bits
O=gpurun_out/ab20; mkdir -p $O
QRT_EVC_LINEAR_COAL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k uniform > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for c in 4 3 2; do
QRT_EVC_LINEAR_COAL=$c python bench.py --no-cpu-baseline --warmup 1 --steps 2 --circuit hea --hamiltonian uniform --terms 1000 > $O/uni_$c.json 2>&1
done
