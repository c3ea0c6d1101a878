#!/bin/bash
O=${OUT:-gpurun_out/r2diag}; mkdir -p $O
for d in 1 0; do
  QRT_EVC_DIAG_ALONE=$d timeout 900 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_diag$d.json 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
