#!/bin/bash
# Round-2 GPU check (run from the repo root under gpurun): full GPU test suite,
# smoke, the default bench line (C3 32q, N=1) and the reference arm.
O=${OUT:-gpurun_out/r2a}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 900 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
timeout 600 python bench.py --impl reference > $O/ref32.json 2> $O/ref32.err
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
