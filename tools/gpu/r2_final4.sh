#!/bin/bash
# Final-tree verification after the EVC latency work: GPU tests, smoke, the default bench line
# (C3 32q), the reference arm, then one ncu --set full capture of a 32-qubit EVC pass.
O=${OUT:-gpurun_out/final4}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --durations=10 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
timeout 900 python bench.py --impl reference > $O/ref32.json 2> $O/ref32.err
ncu --clock-control none --set full --import-source on -k regex:coset_pipe_kernel -s 20 -c 1 -o $O/coset32 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_coset.log 2>&1
echo rc=$? >> $O/ncu_coset.log
