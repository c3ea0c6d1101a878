# scratch A/B script for gpurun (edited per experiment)
O=gpurun_out/ab6; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --warmup 1 --steps 2 > $O/fold.json 2>&1
python tools/gate_sweep.py > $O/sweep.txt 2>&1
