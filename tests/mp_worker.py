"""Multi-process worker (one process per GPU) for tests/test_gpu_multi.py.

Launched by torch.distributed.run; every rank owns p/world PEs of a
distributed state, QRs move amplitudes between GPUs over NVLink (CUDA IPC
peer stores) and EVC partials are gathered with NCCL.  Rank 0 checks the
result against the CPU oracle and prints one JSON line.
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2410_04252_b200 as qb  # noqa: E402
from oracle import cpu  # noqa: E402


def main():
    rank, world, dev = qb.init_distributed()
    import torch.distributed as dist

    results = {}
    cases = [(10, 8, 1, "0"), (14, 6, 2, "0"), (16, 4, 1, "0"), (14, 6, 2, "1"), (16, 4, 1, "1"), (14, 4, 1, "wide")]
    for n, layers, ppr, mode in cases:
        # QRT_QR_INPLACE is read at state creation: "1" = in-place QR (one
        # buffer per PE, pairwise NVLink swap), "0" = push / fused pull
        os.environ["QRT_QR_INPLACE"] = "1" if mode == "1" else "0"
        p = world * ppr
        circuit = qb.gen_gatefabric(n, layers, 3, True)
        if mode == "wide":
            # an 8-qubit gate between GateFabric layers: after a fused QR the
            # wide pass writes the spare buffer peers may still be reading
            ops = list(circuit.operators)
            half = len(ops) // 2
            wide = qb.make_gate(half, [7, 0, 3, 1, 6, 2, 5, 4], qb.random_unitary(8, 77))
            ops = [qb.make_gate(i, list(op.targets), op.payload) for i, op in enumerate(ops[:half])] + [wide] + \
                  [qb.make_gate(half + 1 + i, list(op.targets), op.payload) for i, op in enumerate(ops[half:])]
            circuit = qb.Circuit(n, ops)
        deps = qb.build_dependency_graph(circuit)
        shape = qb.ClusterShape.flat(p)
        terms = qb.gen_synthetic_jw(n, 9, 8)
        for name, fn in (("flat", qb.flat_tiling), ("adhoc", qb.adhoc_schedule)):
            name = f"{name}:{mode}"
            sched = fn(circuit, deps, shape)
            plan = qb.plan_evc(terms, n, shape, True)
            st = qb.init_state(n, shape)
            assert qb.state_mode(st)["inplace_qr"] == (mode == "1")
            qb.run_qsu(st, circuit, sched)
            mine = {pe: st.sub_of(pe) for pe in range(st.pe_begin(), st.pe_begin() + st.pe_count())}
            layout_pos = list(st.layout.pos_of)
            energy = qb.expectation(st, plan, terms)
            norm = st.norm()
            # oracle on every rank (cheap at these sizes)
            sub, lay, moved = cpu.run_qsu(n, p, circuit, sched)
            assert lay.pos_of == layout_pos
            err = max(float(np.max(np.abs(mine[pe] - sub[pe]))) for pe in mine)
            # oracle energy: canonical QSU state, plan executed from the identity layout
            psi = cpu.flatten(sub, lay.qubit_at).reshape(p, -1).copy()
            olay = cpu.Layout(n, p)
            lay_obj = qb.QubitLayout.identity(n, shape)
            partial = np.zeros(p, dtype=complex)
            for tile in plan.tiles:
                if lay_obj.local_set() != tile.local_qubits:
                    ev = qb.make_qr_event(lay_obj, tile.local_qubits)
                    cpu.perform_qr(psi, olay.dest_for(ev.after.pos_of))
                    olay.adopt(ev.after.pos_of)
                    lay_obj = ev.after
                masked = [cpu.mask_term(terms[i].letters, olay.pos_of, olay.nl) for i in tile.terms]
                partial += cpu.expectation_tile(psi, masked, [terms[i].coeff for i in tile.terms])
            want = complex(sum(partial))
            results[f"{name}:n{n}:p{p}"] = {
                "amp_err": err, "energy": energy.real, "oracle": want.real,
                "energy_err": abs(energy - want), "norm": norm, "qr": len(st.qr_log),
                "moved_ok": [m for _, m in st.qr_log][:len(moved)] == moved,
            }
    gathered = [None] * world
    dist.all_gather_object(gathered, results)
    if rank == 0:
        worst_amp = max(v["amp_err"] for r in gathered for v in r.values())
        worst_e = max(v["energy_err"] for r in gathered for v in r.values())
        ok = worst_amp <= 1e-12 and worst_e <= 1e-10 and all(v["moved_ok"] for r in gathered for v in r.values())
        print(json.dumps({"world": world, "ok": ok, "worst_amp_err": worst_amp, "worst_energy_err": worst_e,
                          "cases": gathered[0]}))
    dist.barrier()
    qb.shutdown_device()


if __name__ == "__main__":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    main()
