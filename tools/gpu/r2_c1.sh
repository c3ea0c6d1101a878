#!/bin/bash
# BASELINE C1 (20 qubits, 4 PEs on one GPU, full JW: --span 0, 19,971 strings) on both arms: the reference arm runs the
# reference's whole evaluate_energy here (measured, n <= --cpu-full-qubits), lazy and eager.
O=${OUT:-gpurun_out/c1}; mkdir -p $O
for s in flat adhoc; do
  timeout 900 python bench.py --qubits 20 --pes-per-gpu 4 --span 0 --schedule $s --steps 10 --warmup 3 > $O/bench20_$s.json 2> $O/bench20_$s.err
  timeout 900 python bench.py --impl reference --qubits 20 --pes-per-gpu 4 --span 0 --schedule $s --steps 1 --warmup 0 > $O/ref20_$s.json 2> $O/ref20_$s.err
done
nproc > $O/nproc.txt
