#!/bin/bash
# One GPU: 30q HEA + 1,000 uniform random Pauli words (GF(2)-linear EVC passes),
# the full-vector-sweep fallback for comparison, and one ncu capture of a linear pass.
OUT=${OUT:-gpurun_out/uni}
mkdir -p "$OUT"
python bench.py --no-cpu-baseline --circuit hea --hamiltonian uniform --terms 1000 > "$OUT/uni1000.json" 2> "$OUT/uni1000.err"
QRT_EVC_LINEAR=0 python bench.py --no-cpu-baseline --circuit hea --hamiltonian uniform --terms 1000 > "$OUT/uni1000_sweep.json" 2> "$OUT/uni1000_sweep.err"
ncu --clock-control none --set full --import-source on -k regex:coset_pipe -s 5 -c 1 -o "$OUT/coset_linear30" \
    python bench.py --no-cpu-baseline --circuit hea --hamiltonian uniform --terms 1000 --steps 1 --warmup 0 > "$OUT/ncu.log" 2>&1
echo done > "$OUT/done"
