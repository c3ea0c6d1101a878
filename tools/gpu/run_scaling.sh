#!/bin/bash
# Multi-GPU measurements on one box (gpurun --gpus 4): multi-process GPU tests,
# the default bench strong-scaled to N = 2 and 4, and the BASELINE configs
# C3 (32q GateFabric at N = 1, 2, 4; lazy vs eager QR at 4) and C4/C5 (34q HEA
# + JW EVC at N = 4); then one single-GPU ncu capture of the EVC pipeline kernel.
OUT=${OUT:-gpurun_out/scale}
mkdir -p "$OUT"
R() { python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2" "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > "$OUT/tests_multi.log" 2>&1; echo "rc=$?" >> "$OUT/tests_multi.log"
R 2 29511 bench.py --gpus 2 > "$OUT/b30_gf_n2.json" 2> "$OUT/b30_gf_n2.err"
R 4 29512 bench.py --gpus 4 > "$OUT/b30_gf_n4.json" 2> "$OUT/b30_gf_n4.err"
R 4 29513 bench.py --gpus 4 --circuit hea > "$OUT/b30_hea_n4.json" 2> "$OUT/b30_hea_n4.err"
python bench.py --qubits 32 --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/b32_gf_flat_n1.json" 2> "$OUT/b32_gf_flat_n1.err"
R 2 29520 bench.py --gpus 2 --qubits 32 --steps 1 --warmup 3 > "$OUT/b32_gf_flat_n2.json" 2> "$OUT/b32_gf_flat_n2.err"
R 4 29521 bench.py --gpus 4 --qubits 32 --steps 1 --warmup 3 > "$OUT/b32_gf_flat_n4.json" 2> "$OUT/b32_gf_flat_n4.err"
R 4 29522 bench.py --gpus 4 --qubits 32 --schedule adhoc --steps 1 --warmup 3 > "$OUT/b32_gf_adhoc_n4.json" 2> "$OUT/b32_gf_adhoc_n4.err"
BENCH_DEBUG=1 R 4 29523 bench.py --gpus 4 --qubits 34 --circuit hea --steps 2 --warmup 3 > "$OUT/b34_hea_n4.json" 2> "$OUT/b34_hea_n4.err"
ncu --clock-control none --set full --import-source on -k regex:coset_pipe -s 10 -c 1 -o "$OUT/coset30" \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > "$OUT/ncu_coset.log" 2>&1
echo done > "$OUT/done"
