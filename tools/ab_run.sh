# scratch A/B: GPU tests + HEA/GF bench lines (EVC share)
O=gpurun_out/ab21; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
python bench.py --no-cpu-baseline --circuit hea > $O/hea.json 2>&1
python bench.py --no-cpu-baseline > $O/gf.json 2>&1
