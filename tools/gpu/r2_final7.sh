#!/bin/bash
# Final tree (PE-sign fold): GPU tests, smoke, default bench line (C3 32q)
O=${OUT:-gpurun_out/final7}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
