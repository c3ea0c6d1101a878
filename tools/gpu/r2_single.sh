#!/bin/bash
# EVC one-group-per-mask table path (QRT_EVC_SINGLE) — parity tests, then same-box A/B at 30 qubits.
O=${OUT:-gpurun_out/single}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_configs.py tests/test_gpu_parity.py -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for rep in 1 2; do
  for v in 0 1; do
    QRT_EVC_SINGLE=$v timeout 600 python bench.py --qubits 30 --steps 3 --warmup 3 --cpu-sample-qubits 12 > $O/gf30_s${v}_$rep.json 2> $O/gf30_s${v}_$rep.err
    QRT_EVC_SINGLE=$v timeout 600 python bench.py --qubits 30 --circuit hea --steps 3 --warmup 3 --cpu-sample-qubits 12 > $O/hea30_s${v}_$rep.json 2> $O/hea30_s${v}_$rep.err
  done
done
OUT=$O/c1 bash tools/gpu/r2_c1.sh
