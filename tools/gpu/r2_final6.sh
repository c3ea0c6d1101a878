#!/bin/bash
# Final tree (byte-offset gathers): GPU tests, smoke, default bench line (C3 32q), reference arm
O=${OUT:-gpurun_out/final6}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
timeout 900 python bench.py --impl reference > $O/ref32.json 2> $O/ref32.err
timeout 600 python bench.py --qubits 30 --circuit hea --steps 3 --warmup 3 > $O/hea30.json 2> $O/hea30.err
