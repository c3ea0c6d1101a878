#!/bin/bash
# EVC kernel iteration: GPU EVC tests, 30q GF/HEA bench lines, uniform 30q, ncu of the pipe kernel
O=${OUT:-gpurun_out/r2evc}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30.json 2>&1
timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 2 --warmup 3 > $O/hea30.json 2>&1
timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 1000 --no-cpu-baseline --steps 2 --warmup 3 > $O/hea30_uni1000.json 2>&1
ncu --clock-control none --set full --import-source on -k regex:coset_pipe -s 10 -c 1 -o $O/coset30 \
    python bench.py --qubits 30 --circuit hea --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_coset.log 2>&1
