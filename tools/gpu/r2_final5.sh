#!/bin/bash
# Final tree: GPU tests + smoke, then same-box A/B of the EVC table placement on JW and uniform-word
# passes (product = compiler placement vs libqrt_early1.so), then the default bench line (C3 32q).
O=${OUT:-gpurun_out/final5}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
P=$PWD/paper_2410_04252_b200
for i in 1 2; do
  for v in base early1; do
    if [ $v = base ]; then L=; else L=$P/libqrt_$v.so; fi
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --no-cpu-baseline --steps 3 --warmup 3 > $O/hea30_${v}_$i.json 2>&1
    LD_PRELOAD=$L timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni30_${v}_$i.json 2>&1
  done
done
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
