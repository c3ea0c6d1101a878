import csv, subprocess, sys
keys = sys.argv[2:] or ['gpu__time_duration.sum','sm__pipe_fp64_cycles_active','l1tex__lsu_writeback_active.avg.pct','l1tex__data_pipe_lsu_wavefronts.avg.pct','smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct','smsp__average_warps_issue_stalled','idc','smsp__pcsamp']
out = subprocess.run(['ncu','-i',sys.argv[1],'--page','raw','--csv'],capture_output=True,text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
for row in r[2:]:
    for h,u,v in zip(hdr,units,row):
        if any(k in h for k in keys) and v not in ('','0'):
            print(h[:95].ljust(95), v, u)
