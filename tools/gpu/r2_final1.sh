#!/bin/bash
# One-GPU round evidence: full GPU suite (incl. the checked build), smoke, the default
# bench line (C3 32q, N=1) + reference arm, launch list, ncu captures of the top kernels.
O=${OUT:-gpurun_out/r2f1}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --durations=20 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
BENCH_DEBUG=1 timeout 1200 python bench.py > $O/bench32.json 2> $O/bench32.err; echo rc=$? >> $O/bench32.err
timeout 900 python bench.py --impl reference > $O/ref32.json 2> $O/ref32.err
NCU="ncu --clock-control none"
timeout 1200 $NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_32q.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:gate_pass -s 20 -c 1 -o $O/gate32 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_gate.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:coset_pipe -s 10 -c 1 -o $O/coset32 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_coset.log 2>&1
# single-process 4 PEs with in-place QR: local swap / exchange launch costs
QRT_QR_INPLACE=1 timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file $O/launches_30q_p4_inplace.csv -k regex:"exchange|local_swap|reorder" \
    python -c "
import sys; sys.path.insert(0,'.')
import paper_2410_04252_b200 as qb
qb.init_device(0,1,0)
n=30; c=qb.gen_gatefabric(n,4*n,1,True); s=qb.flat_tiling(c,qb.build_dependency_graph(c),qb.ClusterShape.flat(4))
st=qb.init_state(n,qb.ClusterShape.flat(4)); qb.run_qsu(st,c,s); print(len(st.qr_log))
" > $O/ncu_inplace.log 2>&1
