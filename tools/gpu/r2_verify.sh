#!/bin/bash
# Final-tree verification on a fresh box: GPU tests, smoke, the default bench line, reference arm.
O=${OUT:-gpurun_out/r2verify3}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --durations=10 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
timeout 900 python bench.py --impl reference > $O/ref32.json 2> $O/ref32.err
