#!/bin/bash
# A/B of the split-coset EVC kernel (QRT_EVC_SPLIT) on the 30q GateFabric and HEA steps + EVC tests
O=${OUT:-gpurun_out/r2evc}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_evc.py tests/test_gpu_parity.py -q -x -k "expectation or evc or energy or coset" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for sp in 1 0; do
  QRT_EVC_SPLIT=$sp timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_split$sp.json 2>&1
  QRT_EVC_SPLIT=$sp timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 2 --warmup 3 > $O/hea30_split$sp.json 2>&1
done
ncu --clock-control none --set full --import-source on -k regex:coset_pipe_split -s 10 -c 1 -o $O/coset_split30 \
    python bench.py --qubits 30 --circuit hea --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_split.log 2>&1
