"""Summarise `ncu --set full` captures (.ncu-rep) into the JSON committed under
profiles/: duration, DRAM bytes, pipe utilisations, occupancy, top stall
reasons, per kernel launch.  Optionally records per-launch DRAM traffic in
profiles/roofline_traffic.json under a bench key (circuit:family:qubits:pes),
which bench.py reports as roofline.traffic.

  python tools/ncu_extract.py rep.ncu-rep [--key gatefabric:gates:30:1 --algo-bytes B] > summary.json
"""
import argparse
import csv
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def summarise(rep):
    res = []
    for vals, units in raw(rep):
        d = {"kernel": vals.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in vals and vals[k] != "":
                d[k] = f"{vals[k]} {units.get(k, '')}".strip()
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v))
                  for k, v in vals.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and v not in ("", "0")}
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        res.append(d)
    return res


def to_bytes(s):
    v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
    return float(v) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--key")
    ap.add_argument("--algo-bytes", type=float)
    ap.add_argument("--traffic-json", default=str(Path(__file__).resolve().parent.parent / "profiles" / "roofline_traffic.json"))
    a = ap.parse_args()
    summ = summarise(a.rep)
    json.dump(summ, sys.stdout, indent=1)
    print()
    if a.key and summ:
        k0 = summ[0]
        traffic = to_bytes(k0["dram__bytes_read.sum"]) + to_bytes(k0["dram__bytes_write.sum"])
        p = Path(a.traffic_json)
        d = json.loads(p.read_text()) if p.exists() else {}
        d[a.key] = {"kernel": k0["kernel"][:60], "dram_bytes_per_launch": traffic,
                    "algorithmic_bytes_per_launch": a.algo_bytes, "source": Path(a.rep).name}
        p.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    main()
