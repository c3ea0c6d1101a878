#!/bin/bash
# Round-2 GPU check (run from the repo root under gpurun): full GPU test suite,
# smoke, then the split-coset EVC A/B.
O=${OUT:-gpurun_out/r2c}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --durations=15 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
for sp in 1 0; do
  QRT_EVC_SPLIT=$sp timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_split$sp.json 2>&1
  QRT_EVC_SPLIT=$sp timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 2 --warmup 3 > $O/hea30_split$sp.json 2>&1
done
ncu --clock-control none --set full --import-source on -k regex:coset_pipe_split -s 10 -c 1 -o $O/coset_split30 \
    python bench.py --qubits 30 --circuit hea --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_split.log 2>&1
