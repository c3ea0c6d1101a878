#!/bin/bash
O=${OUT:-gpurun_out/r2chk}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
QRT_QR_INPLACE=1 timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file $O/launches_30q_p4_inplace.csv -k regex:"exchange|local_swap|reorder" \
    python -c "
import sys; sys.path.insert(0,'.')
import paper_2410_04252_b200 as qb
qb.init_device(0,1,0)
n=30; c=qb.gen_gatefabric(n,4*n,1,True); s=qb.flat_tiling(c,qb.build_dependency_graph(c),qb.ClusterShape.flat(4))
st=qb.init_state(n,qb.ClusterShape.flat(4)); qb.run_qsu(st,c,s); print(len(st.qr_log))
" > $O/ncu_inplace.log 2>&1
