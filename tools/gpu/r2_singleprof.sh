#!/bin/bash
# ncu source-level capture of one Jordan-Wigner EVC pass (coset_pipe_kernel, QRT_EVC_SINGLE path) at 30q
O=${OUT:-gpurun_out/singleprof}; mkdir -p $O
ncu --clock-control none --set full --import-source on -k regex:coset_pipe_kernel -s 20 -c 1 -o $O/coset_single30 \
    python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu.log 2>&1
echo rc=$? >> $O/ncu.log
