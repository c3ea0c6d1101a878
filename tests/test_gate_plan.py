"""Host-only checks of the gate-pass planner (csrc/qrt_gates.cu, plan_gates)
through qrt_gate_plan_info: no device needed.

The planner re-applies the reference's tile construction
(qsu_scheduler.cpp:37-60) at SM level; these tests pin how it packs the
BASELINE circuits: GateFabric's dense 4-qubit blocks into shared-memory DMMA
passes, the hardware-efficient ansatz (RY, RZ, CZ) into register-resident
light passes with RY.RZ fused on the host and CZ handled as signs.
"""
import ctypes as C

import numpy as np
import pytest


def _arrays(circuit, nl):
    arity, pos, mats, flags = [], [], [], []
    for op in circuit.operators:
        if any(q >= nl for q in op.targets):
            continue
        U = np.asarray(op.payload)
        diag = np.count_nonzero(U - np.diag(np.diag(U))) == 0
        arity.append(len(op.targets))
        pos.extend(op.targets)
        flags.append(1 if diag else 0)
        vals = np.diag(U) if diag else U.reshape(-1)
        for v in vals:
            mats.extend([v.real, v.imag])
    return (np.array(arity, np.int32), np.array(pos, np.int32), np.array(mats, np.float64),
            np.array(flags, np.uint32))


def plan_info(qb, circuit, nl):
    lib = qb.load_libqrt()
    a, p, m, f = _arrays(circuit, nl)
    out = [C.c_int() for _ in range(4)]
    IP = C.POINTER(C.c_int)
    rc = lib.qrt_gate_plan_info(nl, len(a), a.ctypes.data_as(IP), p.ctypes.data_as(IP),
                                m.ctypes.data_as(C.POINTER(C.c_double)), f.ctypes.data_as(C.POINTER(C.c_uint)),
                                *[C.byref(o) for o in out])
    assert rc == 0, lib.qrt_last_error()
    return {"passes": out[0].value, "light": out[1].value, "stages": out[2].value, "fused": out[3].value,
            "gates": len(a)}


def test_gatefabric_30q_dmma_passes(qb):
    c = qb.gen_gatefabric(30, 120, 1, True)
    info = plan_info(qb, c, 30)
    assert info["gates"] == 1680 and info["light"] == 0 and info["fused"] == 0
    assert 300 <= info["passes"] <= 420, info  # ~4.4 dense 4-qubit blocks per HBM pass


def test_hea_30q_light_passes(qb):
    c = qb.gen_hea(30, 20, 1, True)
    info = plan_info(qb, c, 30)
    assert info["fused"] == 600  # RZ folded into the RY before it, every qubit, every layer
    assert info["light"] == info["passes"] and info["passes"] <= 40, info
    assert info["passes"] <= info["stages"] <= 4 * info["passes"]


def test_knobs_disable_light_and_fusion(qb, monkeypatch):
    c = qb.gen_hea(20, 6, 3, True)
    monkeypatch.setenv("QRT_LIGHT", "0")
    monkeypatch.setenv("QRT_FUSE_1Q", "0")
    info = plan_info(qb, c, 20)
    assert info["light"] == 0 and info["fused"] == 0 and info["passes"] > 0


@pytest.mark.parametrize("nl,light", [(11, False), (12, True), (13, True)])
def test_light_needs_a_full_tile(qb, nl, light):
    c = qb.gen_hea(nl, 3, 2, True)
    info = plan_info(qb, c, nl)
    assert (info["light"] > 0) == light


def test_random_mixes_plan(qb):
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(12, 24))
        ops = []
        for i in range(int(rng.integers(1, 200))):
            k = int(rng.integers(1, 5))
            t = [int(x) for x in rng.choice(n, size=k, replace=False)]
            if rng.random() < 0.4:
                U = np.diag(np.where(rng.random(1 << k) < 0.5, -1.0, 1.0)).astype(complex)
            else:
                U = qb.random_unitary(k, int(rng.integers(1 << 62)))
            ops.append(qb.make_gate(i, t, U))
        info = plan_info(qb, qb.Circuit(n, ops), n)
        assert 1 <= info["passes"] <= len(ops)
