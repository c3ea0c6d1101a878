# scratch A/B script for gpurun (edited per experiment)
O=gpurun_out/ab17; mkdir -p $O
QRT_GAUSS=2 QRT_GATE_REGS=168 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --warmup 1 --steps 2 > $O/base.json 2>&1
QRT_GAUSS=2 QRT_GATE_REGS=168 python bench.py --no-cpu-baseline --warmup 1 --steps 2 > $O/hoist.json 2>&1
QRT_GATE_REGS=168 python bench.py --no-cpu-baseline --warmup 1 --steps 2 > $O/r168.json 2>&1
