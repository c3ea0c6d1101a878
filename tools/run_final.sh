#!/bin/bash
# Round-end verification on one GPU: GPU parity tests, smoke, then the
# profiling pass (bench lines, launch lists, ncu captures).
OUT=${OUT:-gpurun_out/final}
mkdir -p "$OUT"
timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/tests_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/tests_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
python bench.py --impl reference --steps 1 --warmup 0 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
OUT=$OUT/prof bash tools/profile_round.sh > "$OUT/prof.log" 2>&1
echo done > "$OUT/done"
