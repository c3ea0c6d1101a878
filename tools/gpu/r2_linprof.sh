#!/bin/bash
# ncu source-level capture of one GF(2)-linear EVC pass (uniform words) and the C5 line at 30q
O=${OUT:-gpurun_out/r2linprof}; mkdir -p $O
timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni4000.json 2>&1
ncu --clock-control none --set full --import-source on -k regex:coset_pipe_kernel -s 20 -c 1 -o $O/coset_lin30 \
    python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu.log 2>&1
