#!/usr/bin/env python
"""One VQE iteration (QSU + QR + EVC) of arXiv 2410.04252 on B200.

Workload (BASELINE.json configs[2], "C3" — the metric is quoted at 32-34
qubits and 32 qubits is the largest config that fits one GPU): GateFabric,
n=32 qubits, layers=4n=128 (1,920 dense 4-qubit blocks, Rng seed 1), lazy
flat_tiling schedule, then EVC of the synthetic Jordan-Wigner Hamiltonian
gen_synthetic_jw(32, 1, max_span=10) (8,994 strings) with diagonalization.
At N GPUs the same 32-qubit state (64 GiB) is sharded 2^g-way (p = N, strong
scaling, C3's "1/2/4/8 B200"); the schedule's QRs move amplitudes over NVLink.
--qubits 30 gives C2, --circuit hea --qubits 34 C4, --hamiltonian uniform C5.

A step = init_state + run_qsu + expectation through the public API
(= evaluate_energy, dist_sim.cpp:357-363).  `value` is the step's device time
(CUDA events on the libqrt stream, max over ranks); `e2e` is the host wall
time of the same public-API step, which includes every host->device copy of
the step's inputs (gate payloads, term masks) and the device->host read of the
per-PE partial sums.  The 16-32 GiB state is far larger than L2, so no flush is
needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_PEAK_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback
# FP64 tensor (DMMA) peak measured on this pool's B200s by tools/microbench_fp64.cu
# (profiles/r1_microbench_fp64.txt: 37.0 TFLOP/s; datasheet 296 TF / 8 = 37).  MEASURED_PEAKS.json
# only carries bf16, which is not the gate kernel's arithmetic.
FP64_TENSOR_PEAK = 37.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--qubits", type=int, default=32,
                    help="32 = C3, the metric's configuration (64 GiB state on one GPU); 30 = C2; 34 = C4/C5")
    ap.add_argument("--circuit", choices=["gatefabric", "hea"], default="gatefabric",
                    help="gatefabric (C2/C3) or the hardware-efficient ansatz (C4)")
    ap.add_argument("--layers", type=int, default=0, help="default 4n for GateFabric (PAPER.md:958), 20 for HEA")
    ap.add_argument("--hamiltonian", choices=["jw", "uniform"], default="jw",
                    help="jw: gen_synthetic_jw(n,1,span); uniform: --terms random words (C5 stress)")
    ap.add_argument("--terms", type=int, default=10000)
    ap.add_argument("--span", type=int, default=10)
    ap.add_argument("--schedule", choices=["flat", "hierarchical", "adhoc"], default="flat")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pes-per-gpu", type=int, default=1,
                    help="PEs per GPU (p = N x this): runs a p-PE schedule (e.g. the p = 8 configs) on fewer GPUs")
    ap.add_argument("--cpu-sample-qubits", type=int, default=24)
    ap.add_argument("--cpu-full-qubits", type=int, default=20,
                    help="up to this size the reference arm runs the whole evaluate_energy (measured, C1)")
    return ap.parse_args()


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices: str):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", devices, f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def workload(qb, args, p):
    n = args.qubits
    if args.circuit == "hea":
        layers = args.layers or 20
        circuit = qb.gen_hea(n, layers, 1, True)
    else:
        layers = args.layers or 4 * n
        circuit = qb.gen_gatefabric(n, layers, 1, True)
    deps = qb.build_dependency_graph(circuit)
    shape = qb.ClusterShape.flat(p)
    sched = {"flat": qb.flat_tiling, "hierarchical": qb.hierarchical_tiling, "adhoc": qb.adhoc_schedule}[args.schedule](
        circuit, deps, shape)
    terms = (qb.gen_synthetic_jw(n, 1, args.span) if args.hamiltonian == "jw"
             else qb.gen_uniform_words(n, args.terms, 2024))
    plan = qb.plan_evc(terms, n, shape, True, 8)
    return n, layers, circuit, sched, terms, plan, shape


def config_of(args, n, layers, n_gates, n_terms, p, qr_qsu=None, qr_evc=None):
    cfg = {30: "C2", 32: "C3", 34: "C4/C5"}.get(n, "custom")
    circ = (f"{cfg} GateFabric {n}q layers={layers} ({n_gates} dense 4q gates, seed 1)" if args.circuit == "gatefabric"
            else f"C4 HEA {n}q depth={layers} ({n_gates} gates: RY dense, RZ/CZ diagonal, seed 1)")
    ham = (f"gen_synthetic_jw({n},1,max_span={args.span})" if args.hamiltonian == "jw"
           else "C5 stress: uniform words IXYZ[Rng(2024).below(4)]")
    sched = {"flat": "lazy (flat_tiling)", "hierarchical": "lazy (hierarchical_tiling)",
             "adhoc": "eager (adhoc_schedule)"}[args.schedule]
    return {"workload": f"{circ} + EVC of {ham} ({n_terms} Pauli strings), {sched} schedule, p={p}",
            "qubits": n, "pes": p, "schedule": args.schedule, "qr_qsu": qr_qsu, "qr_evc": qr_evc,
            "l2": "inputs larger than L2 (state 16 B x 2^n)", "parallelism": f"state sharded {p}-way"}


def reference_counts(args, p):
    """Gate, string and QR counts of the full-size workload from the reference
    itself (oracle/_ref): its generators, its scheduler (qsu_scheduler.cpp) and
    its EVC planner (evc_scheduler.cpp); the EVC QRs are re-derived from the
    post-QSU layout exactly as expectation() does (dist_sim.cpp:268-271)."""
    from oracle import ref as R

    n = args.qubits
    if args.circuit == "hea":
        layers = args.layers or 20
        circ = R.Circuit.hea(n, layers, 1)
    else:
        layers = args.layers or 4 * n
        circ = R.Circuit.gatefabric(n, layers, 1, False)
    arity, _, _ = circ.export()
    per_arity = [int((arity == a).sum()) for a in (1, 2, 3, 4)]
    terms = R.Terms.jw(n, 1, args.span) if args.hamiltonian == "jw" else R.Terms.uniform(n, args.terms, 2024)
    ks = []
    qr_qsu = qr_evc = 0
    nl = n - (p.bit_length() - 1)
    locals_ = (1 << nl) - 1
    if p > 1:
        d = circ.schedule(args.schedule, p)
        for ev in d["events"]:
            new = sum(1 << q for q, pos in enumerate(ev["after_pos_of"]) if pos < nl)
            ks.append(bin(new & ~locals_).count("1"))
            locals_ = new
        qr_qsu = len(ks)
        plan = terms.plan(n, p, 0, 0, True, 8)
        for tile in plan["plan"]["tiles"]:
            new = sum(1 << q for q in tile["local_qubits"])
            if new != locals_:
                ks.append(bin(new & ~locals_).count("1"))
                locals_ = new
                qr_evc += 1
    return {"n": n, "layers": layers, "per_arity": per_arity, "n_gates": circ.m, "n_terms": terms.count,
            "qr_k": ks, "qr_qsu": qr_qsu, "qr_evc": qr_evc}


def cpu_baseline(args, p, counts=None):
    """The reference's own CPU path (oracle/_ref = the unmodified reference
    library) on SURVEY.md §8d's bounded sample: at n_s qubits and the same p,
    the first 16 gates of each arity through apply_gate_narrow, the first 64
    strings through expectation, one perform_qr per k — then extrapolated
    linearly to the full workload (per-gate / per-string / per-QR cost scales as
    2^n at fixed k).  Threads: workers = nproc, of which the reference itself
    uses min(workers, p) (dist_sim.cpp:25); perform_qr is single-threaded.
    Never imports the product."""
    from oracle import ref as R

    if not R.available():
        return None
    nproc = os.cpu_count() or 1
    counts = counts or reference_counts(args, p)
    n = counts["n"]
    if n <= args.cpu_full_qubits:
        # small enough to run the reference's whole evaluate_energy (dist_sim.cpp:357-363):
        # measured, not extrapolated (C1: 20 qubits, 4 PEs, full JW ~ 40 s with 4 workers)
        layers = counts["layers"]
        circ = R.Circuit.hea(n, layers, 1) if args.circuit == "hea" else R.Circuit.gatefabric(n, layers, 1, True)
        terms = R.Terms.jw(n, 1, args.span) if args.hamiltonian == "jw" else R.Terms.uniform(n, args.terms, 2024)
        t0 = time.time()
        _e, a_qr, b_qr = R.evaluate_energy(circ, terms, args.schedule, p, 0, 0, True, nproc)
        wall = time.time() - t0
        return {"value": wall, "unit": "s", "cores": min(nproc, p), "nproc": nproc, "workers": nproc,
                "kind": "reference", "counts": counts,
                "sample": f"the reference's full evaluate_energy (oracle/_ref) at n={n}, p={p}, workers={nproc} "
                          f"(it uses min(workers, p) = {min(nproc, p)} threads; QR 1 thread): measured, "
                          f"{a_qr} + {b_qr} QRs"}
    ns = min(args.cpu_sample_qubits, n)
    if args.circuit == "hea":
        circ = R.Circuit.hea(ns, 1, 1)
    else:
        circ = R.Circuit.gatefabric(ns, 4, 1, True)
    terms = R.Terms.jw(ns, 1, args.span) if args.hamiltonian == "jw" else R.Terms.uniform(ns, 4096, 2024)
    t0 = time.time()
    g, t, q = R.time_prefix(circ, terms, p, nproc, 16, 64)
    wall = time.time() - t0
    scale = float(1 << (n - ns))
    gates_s = sum(c * s for c, s in zip(counts["per_arity"], g)) * scale
    evc_s = counts["n_terms"] * t * scale
    qr_s = sum(q[k - 1] for k in counts["qr_k"]) * scale
    per_iter = gates_s + evc_s + qr_s
    return {"value": per_iter, "unit": "s", "cores": min(nproc, p), "nproc": nproc, "workers": nproc,
            "kind": "reference",
            "phases_s": {"gates": gates_s, "evc": evc_s, "qr": qr_s},
            "counts": counts,
            "sample": f"reference dist_sim (oracle/_ref): first 16 gates per arity (apply_gate_narrow), 64 strings "
                      f"(expectation), one perform_qr per k at n={ns}, p={p}, workers={nproc} (the reference uses "
                      f"min(workers, p) = {min(nproc, p)} threads; QR 1 thread); {wall:.1f} s of CPU work. "
                      f"Per-gate s by arity {[round(x, 4) for x in g]}, per-string {t:.4g} s, per-QR s by k "
                      f"{[round(x, 4) for x in q]}; scaled by 2^{n - ns} to {counts['n_gates']} gates + "
                      f"{counts['n_terms']} strings + {len(counts['qr_k'])} QRs (extrapolated, linear in 2^n)"}


def loaded_native():
    """In-tree shared objects mapped into this process (reference arm: oracle/_ref only)."""
    try:
        maps = open("/proc/self/maps").read().splitlines()
    except OSError:
        return []
    return sorted({m.split()[-1] for m in maps if m.endswith(".so") and str(ROOT) in m})


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref as R

    p = max(1, world) * args.pes_per_gpu
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqrtile_ref.so not built"}))
        return 0
    counts = reference_counts(args, p)
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        base = cpu_baseline(args, p, counts)
        if i >= args.warmup:
            vals.append(base["value"])
    v = statistics.median(vals)
    base["value"] = v
    line = {"metric": "VQE iteration time (QSU+EVC)", "value": v, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_of(args, counts["n"], counts["layers"], counts["n_gates"], counts["n_terms"], p,
                                counts["qr_qsu"], counts["qr_evc"]),
            "cpu_baseline": base, "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_so_loaded": loaded_native()}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import numpy as np
    import torch

    import paper_2410_04252_b200 as qb

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    qb.init_distributed(device=local)
    torch.cuda.set_device(local)
    p = world * args.pes_per_gpu
    n, layers, circuit, sched, terms, plan, shape = workload(qb, args, p)
    n_gates, n_terms = circuit.size(), len(terms)
    hbm_peak, peak_kind = peaks()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(profile=False):
        t0 = time.perf_counter()
        st = qb.init_state(n, shape)
        if profile:
            st.profile(True)
        stream = torch.cuda.ExternalStream(st.stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        qb.run_qsu(st, circuit, sched)
        qr_qsu = len(st.qr_log)
        energy = qb.expectation(st, plan, terms).real
        e1.record(stream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        dev = e0.elapsed_time(e1) / 1e3
        return st, energy, dev, wall, qr_qsu

    # one sampler on rank 0 for every GPU of the job, started before the
    # warm-up so its start-up (driver queries) is over before the timed steps
    class _NoClocks:
        def stop(self):
            return None

    clocks = Clocks(",".join(str(i) for i in range(world))) if rank == 0 else _NoClocks()
    # warm-up; the last warm-up step is the profiled one (per-kernel-family CUDA
    # events for the roofline), so no extra step is needed after the timed ones
    stats = None
    for i in range(args.warmup):
        st, energy, _, _, _ = step(profile=(i == args.warmup - 1))
        if i == args.warmup - 1:
            stats = st.stats()
            inplace_qr = qb.state_mode(st)["inplace_qr"]
        del st
    barrier()
    torch.cuda.synchronize()
    devs, walls, launches = [], [], 0
    for _ in range(args.steps):
        st, energy, dev, wall, qr_qsu = step()
        devs.append(dev)
        walls.append(wall)
        launches += sum(v["launches"] for v in st.stats().values())
        qr_total = len(st.qr_log)
        del st
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if os.environ.get("BENCH_DEBUG"):
        print(f"rank {rank}: step device s {devs}, wall s {walls}", file=sys.stderr)
    dev_t = max_over_ranks(statistics.mean(devs))
    wall_t = max_over_ranks(statistics.mean(walls))

    if stats is None:  # --warmup 0: profile one extra untimed step
        st, _, _, _, _ = step(profile=True)
        stats = st.stats()
        inplace_qr = qb.state_mode(st)["inplace_qr"]
        del st
    g, qr, pa, xf = stats["gates"], stats["qr"], stats["pauli"], stats["qr_xfer"]
    fam_kernel = {"gates": ("gate_pass_kernel (DMMA fp64 tensor, dense 3/4-qubit gates)" if args.circuit == "gatefabric"
                            else "light_pass_kernel (register-resident 1q/2q/diagonal runs)"),
                  "pauli": "coset_pass_kernel (EVC, 5-qubit register cosets)"}
    try:  # DRAM bytes per launch from the committed `ncu --set full` captures (same n, p, circuit)
        tr = json.loads((ROOT / "profiles" / "roofline_traffic.json").read_text())
    except Exception:
        tr = {}

    def family(name, st, bytes_unit):
        """Achieved vs peak for one kernel family from the profiled step's CUDA events.
        bytes: algorithmic HBM bytes (gates: 32 B x amplitudes per pass, EVC: 16 B per pass);
        flops: reference-equivalent fp64 flops (8*2^k per amplitude per dense k-qubit gate,
        8 per amplitude per Pauli string)."""
        if st["launches"] == 0 or st["ms"] <= 0:
            return None
        sec = st["ms"] / 1e3
        gbs = st["bytes"] / sec / 1e9
        tf = st["flops"] / sec / 1e12
        key = f"{args.circuit}:{name}:{n}:{p}"
        traffic = tr.get(key, {}).get("dram_bytes_per_launch")
        return {"kernel": fam_kernel.get(name, name), "ms": st["ms"], "launches": st["launches"],
                "avg_launch_ms": st["ms"] / st["launches"], "algorithmic_bytes_per_launch": st["bytes"] / st["launches"],
                "algorithmic_flops_per_launch": st["flops"] / st["launches"], "hbm_gbs": gbs,
                "hbm_frac": gbs / hbm_peak, "fp64_tflops_ref_equiv": tf, "fp64_frac": tf / FP64_TENSOR_PEAK,
                "traffic": traffic}

    fams = {k: v for k, v in (("gates", family("gates", g, 32)), ("pauli", family("pauli", pa, 16))) if v}
    top = max(fams, key=lambda k: fams[k]["ms"])
    f = fams[top]
    if top == "gates" and args.circuit == "gatefabric":
        # dense 4-qubit blocks on the fp64 tensor pipe: flop-bound (SURVEY.md section 7 hard parts)
        roof = {"bound": "tensor", "achieved": f["fp64_tflops_ref_equiv"], "peak": FP64_TENSOR_PEAK, "unit": "TFLOP/s",
                "frac": f["fp64_frac"], "peak_kind": "builder-measured fp64 DMMA (tools/microbench_fp64.cu, profiles/r1_microbench_fp64.txt; not in MEASURED_PEAKS.json)"}
        # `achieved` counts the reference's algorithmic flops.  The Gauss-form
        # kernel executes 3 real 16x16 products + 1 DADD per amplitude instead of the
        # 16 complex MACs: 98 of 128 flop-slots on the shared fp64 datapath.
        gauss = os.environ.get("QRT_GAUSS", "1") != "0"
        ex = f["fp64_tflops_ref_equiv"] * (98.0 / 128.0 if gauss else 1.0)
        roof.update({"frac_note": "achieved counts the reference algorithm's 8*2^k flops per amplitude per dense "
                                  "k-qubit gate (SURVEY.md 8d); the kernel's Gauss form needs 98/128 of them, so frac "
                                  "can exceed 1 - executed_frac is the fp64 datapath occupancy",
                     "executed_tflops": ex, "executed_frac": ex / FP64_TENSOR_PEAK,
                     "executed_note": "fp64 datapath slots actually issued (Gauss form: 3 DMMA products + 1 DADD "
                                      "per amplitude = 98/128 of the reference flops)" if gauss else "real form"})
    else:
        # light passes and EVC passes: one HBM round trip (gates) / read (EVC) per pass
        roof = {"bound": "hbm", "achieved": f["hbm_gbs"], "peak": hbm_peak, "unit": "GB/s", "frac": f["hbm_frac"],
                "peak_kind": peak_kind}
    roof.update({"kernel": f["kernel"], "traffic": f["traffic"], "avg_launch_ms": f["avg_launch_ms"],
                 "algorithmic_bytes_per_launch": f["algorithmic_bytes_per_launch"],
                 "algorithmic_flops_per_launch": f["algorithmic_flops_per_launch"], "families": fams})
    mat_bytes = sum(16 * (1 << (2 * op.arity())) for op in circuit.operators)
    term_bytes = 8 * 5 * n_terms
    d2h = 16 * p * max(1, len(plan.tiles))
    if rank != 0:
        return 0
    line = {
        "metric": "VQE iteration time (QSU+EVC)", "value": dev_t, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_t * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, n, layers, n_gates, n_terms, p, qr_qsu, qr_total - qr_qsu),
        "energy": energy,
        "e2e": {"value": wall_t, "unit": "s", "h2d_bytes_per_step": mat_bytes + term_bytes, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches // max(1, args.steps),
        "clocks": clk,
        "roofline": roof,
        "phases_ms": {"gates": g["ms"], "qr": qr["ms"], "pauli": pa["ms"], "misc": stats["misc"]["ms"],
                      "qr_exchange_kernels": xf["ms"], "qr_barriers": qr["ms"] - xf["ms"],
                      "gate_passes": g["launches"], "qr_launches": qr["launches"], "pauli_passes": pa["launches"],
                      "qr_nvlink_gbs_incl_barriers": (qr["bytes"] / (qr["ms"] / 1e3) / 1e9) if qr["ms"] > 0 else None,
                      "qr_nvlink_gbs": (xf["bytes"] / (xf["ms"] / 1e3) / 1e9) if xf["ms"] > 0 else None,
                      "qr_mode": "in-place (pairwise swap)" if inplace_qr else "push / fused pull (two buffers)"},
    }
    line["native_so_loaded"] = loaded_native()
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, p)
    print(json.dumps(line))
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
