"""Command-line driver with the reference's sub-commands, flags, text formats
and report keys (proj/tools/qrtile_cli.cpp:46-106, proj/src/report.cpp:80-280),
running `simulate` / `evc` on the B200 backend:

  python -m paper_2410_04252_b200.cli schedule --fixture gatefabric-fig6
  python -m paper_2410_04252_b200.cli simulate --circuit c.txt --p 4 --verify --out state.bin
  python -m paper_2410_04252_b200.cli evc --fixture jw12 --p 4
  python -m paper_2410_04252_b200.cli bench --sweep-n 16,20 --layers 4

Exit codes as in the reference (qrtile_cli.cpp:94-105, report.cpp:181,254):
0 success, 1 a requested verification failed, 2 usage / input errors.
Options may also come from a `--config` file of `key=value` lines (keys are
the long flag names); flags given on the command line win.

`--verify` compares against a dense state vector (n <= 14, the reference's
own bar, dist_sim.cpp:302-355 / kOracleMaxQubits); it is a report check and
never feeds a result.
"""
from __future__ import annotations

import argparse
import io
import json
import sys
import time

import numpy as np

import paper_2410_04252_b200 as qb

SCHEDULERS = ("flat", "hierarchical", "adhoc")


# ------------------------------------------------------------------ text formats

def _tokenize(text):
    """models.cpp:285-301: '#' starts a comment; blank lines are skipped."""
    for number, raw in enumerate(text.splitlines(), start=1):
        toks = raw.split("#", 1)[0].split()
        if toks:
            yield number, toks


def _int(number, tok):
    try:
        return int(tok)
    except ValueError:
        raise qb.ParseError(f"line {number}: expected an integer, got '{tok}'") from None


def _float(number, tok):
    try:
        return float(tok)
    except ValueError:
        raise qb.ParseError(f"line {number}: expected a number, got '{tok}'") from None


def _letter_qubit(number, tok):
    if len(tok) < 2 or tok[0] not in "XYZ":
        raise qb.ParseError(f"line {number}: expected <letter><qubit>, got '{tok}'")
    return tok[0], _int(number, tok[1:])


def parse_circuit(text):
    """parse_circuit, models.cpp:343-410: `n <count>`, `G <id> <q>...`, `P <id> <L><q>...`."""
    raw, declared, maxq = [], -1, -1
    for number, t in _tokenize(text):
        if t[0] == "n":
            if len(t) != 2:
                raise qb.ParseError(f"line {number}: expected 'n <count>'")
            declared = _int(number, t[1])
            continue
        if t[0] not in ("G", "P"):
            raise qb.ParseError(f"line {number}: expected 'G' or 'P' line, got '{t[0]}'")
        if len(t) < 2:
            raise qb.ParseError(f"line {number}: missing operator id")
        op = {"line": number, "kind": t[0], "id": _int(number, t[1])}
        if t[0] == "G":
            if len(t) < 3:
                raise qb.ParseError(f"line {number}: gate needs at least one target")
            op["qubits"] = [_int(number, x) for x in t[2:]]
            maxq = max([maxq] + op["qubits"])
        else:
            op["pauli"] = [_letter_qubit(number, x) for x in t[2:]]
            maxq = max([maxq] + [q for _, q in op["pauli"]])
        raw.append(op)
    n = declared if declared >= 0 else maxq + 1
    if n <= 0:
        raise qb.ParseError("cannot determine qubit count")
    ops = []
    for i, op in enumerate(raw):
        if op["id"] != i:
            raise qb.ParseError(f"line {op['line']}: operator ids must be dense and in file order")
        if op["kind"] == "G":
            for q in op["qubits"]:
                if q < 0 or q >= n:
                    raise qb.IndexError(f"line {op['line']}: qubit {q} out of range")
            ops.append(qb.make_gate(op["id"], op["qubits"]))
        else:
            letters = ["I"] * n
            for ch, q in op["pauli"]:
                if q < 0 or q >= n:
                    raise qb.IndexError(f"line {op['line']}: qubit {q} out of range")
                letters[q] = ch
            ops.append(qb.make_pauli_op(op["id"], "".join(letters)))
    c = qb.Circuit(n, ops)
    c.validate()
    return c


def parse_hamiltonian(text):
    """parse_hamiltonian, models.cpp:429-470: `n <count>`, `<re> <im> <L><q>...`."""
    raw, declared, maxq = [], -1, -1
    for number, t in _tokenize(text):
        if t[0] == "n":
            if len(t) != 2:
                raise qb.ParseError(f"line {number}: expected 'n <count>'")
            declared = _int(number, t[1])
            continue
        if len(t) < 2:
            raise qb.ParseError(f"line {number}: expected '<re> <im> [letters...]'")
        term = {"line": number, "c": complex(_float(number, t[0]), _float(number, t[1])),
                "pauli": [_letter_qubit(number, x) for x in t[2:]]}
        maxq = max([maxq] + [q for _, q in term["pauli"]])
        raw.append(term)
    n = declared if declared >= 0 else maxq + 1
    if n <= 0 and raw:
        raise qb.ParseError("cannot determine qubit count")
    n = max(n, 1)
    terms = []
    for rt in raw:
        letters = ["I"] * n
        for ch, q in rt["pauli"]:
            if q < 0 or q >= n:
                raise qb.IndexError(f"line {rt['line']}: qubit {q} out of range")
            letters[q] = ch
        terms.append(qb.PauliTerm(rt["c"], "".join(letters)))
    return terms, n


def serialize_circuit(circuit):
    """serialize_circuit, models.cpp:412-427."""
    lines = [f"n {circuit.n}"]
    for op in circuit.operators:
        if op.is_gate:
            lines.append(f"G {op.id} " + " ".join(str(q) for q in op.targets))
        else:
            lines.append(f"P {op.id} " + " ".join(f"{op.letters[q]}{q}" for q in op.targets))
    return "\n".join(lines) + "\n"


def serialize_hamiltonian(terms, n):
    """serialize_hamiltonian, models.cpp:472-487 (%.17g coefficients)."""
    lines = [f"n {n}"]
    for t in terms:
        parts = [f"{t.coeff.real:.17g}", f"{t.coeff.imag:.17g}"]
        parts += [f"{ch}{q}" for q, ch in enumerate(t.letters) if ch != "I"]
        lines.append(" ".join(parts))
    return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ configuration

def _weights(text):
    if not text:
        return qb.CostWeights()
    if "," not in text:
        raise qb.ConfigError("--weights expects wi,we")
    a, b = text.split(",", 1)
    try:
        w = qb.CostWeights(float(a), float(b))
    except ValueError:
        raise qb.ConfigError("--weights expects two numbers") from None
    w.validate()
    return w


def _resolve_shape(cfg, fallback):
    """RunConfig::resolve_shape, report.cpp:75-90."""
    if cfg.nodes > 0 or cfg.gpn > 0:
        if cfg.nodes <= 0 or cfg.gpn <= 0:
            raise qb.ConfigError("--nodes and --gpn must be given together")
        s = qb.ClusterShape.two_level(cfg.nodes, cfg.gpn)
        if cfg.p > 0 and cfg.p != s.p:
            raise qb.ConfigError("--p disagrees with --nodes * --gpn")
        s.validate()
        return s
    if cfg.p > 0:
        s = qb.ClusterShape.flat(cfg.p)
        s.validate()
        return s
    return fallback


def _config_echo(cfg, shape):
    return {"p": shape.p, "n_node": shape.n_node, "n_gpn": shape.n_gpn, "scheduler": cfg.scheduler,
            "seed": cfg.seed, "weights": [cfg.w.w_intra, cfg.w.w_inter], "diagonalize": cfg.diagonalize != "off",
            "workers": cfg.workers}


def _load_circuit(cfg, need_payloads):
    if cfg.fixture:
        return qb.fixture_circuit(cfg.fixture, cfg.seed), qb.fixture_shape(cfg.fixture)
    if cfg.circuit:
        try:
            text = open(cfg.circuit).read()
        except OSError:
            raise qb.ConfigError(f"cannot open circuit file: {cfg.circuit}") from None
        c = parse_circuit(text)
        if need_payloads:
            c = qb.seed_payloads(c, cfg.seed)
        return c, qb.ClusterShape.flat(1)
    raise qb.ConfigError("no circuit input: use --fixture or --circuit")


def _load_hamiltonian(cfg):
    if cfg.hamiltonian:
        try:
            text = open(cfg.hamiltonian).read()
        except OSError:
            raise qb.ConfigError(f"cannot open Hamiltonian file: {cfg.hamiltonian}") from None
        return parse_hamiltonian(text)
    if cfg.fixture:
        return qb.fixture_hamiltonian(cfg.fixture)
    raise qb.ConfigError("no Hamiltonian input: use --fixture or --hamiltonian")


def _emit(cfg, out, text):
    if cfg.out:
        try:
            with open(cfg.out, "w") as f:
                f.write(text)
        except OSError:
            raise qb.ConfigError(f"cannot write output file: {cfg.out}") from None
    else:
        out.write(text)


def _dumps(obj):
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"  # nlohmann::json::dump(2): sorted keys


def _scheduler(name, circuit, deps, shape):
    fn = {"flat": qb.flat_tiling, "hierarchical": qb.hierarchical_tiling, "adhoc": qb.adhoc_schedule}.get(name)
    if fn is None:
        raise qb.ConfigError(f"unknown scheduler: {name}")
    return fn(circuit, deps, shape)


def _metrics(sched, weights, ms):
    c = qb.count_qrs(sched)
    return {"n_qr": c.total, "n_intra": c.intra, "n_inter": c.inter, "cost": qb.qr_cost(c, weights),
            "tiles": len(sched.tiles), "tile_sizes": [len(t.gates) for t in sched.tiles], "sched_time_ms": ms}


# ------------------------------------------------------------------ dense check (--verify only)

def _dense_apply(psi, n, op):
    """dense_oracle_apply (dist_sim.cpp:302-330): matrix bit j <-> targets[j]."""
    if not op.is_gate:
        return psi
    t = list(op.targets)
    k = len(t)
    U = np.asarray(op.payload).reshape(1 << k, 1 << k)
    axes = [n - 1 - q for q in reversed(t)]  # tensor axis of qubit q is n-1-q; matrix bit j <-> t[j]
    v = np.moveaxis(psi.reshape([2] * n), axes, list(range(k))).reshape(1 << k, -1)
    v = U @ v
    return np.moveaxis(v.reshape([2] * n), list(range(k)), axes).reshape(-1)


def _dense_expectation(psi, n, terms):
    """dense_oracle_expectation (dist_sim.cpp:332-355)."""
    idx = np.arange(1 << n, dtype=np.int64)
    total = 0j
    for term in terms:
        x = sum(1 << q for q, ch in enumerate(term.letters) if ch in "XY")
        zy = sum(1 << q for q, ch in enumerate(term.letters) if ch in "ZY")
        ny = sum(1 for ch in term.letters if ch == "Y")
        par = np.array([bin(v).count("1") & 1 for v in (idx & zy)], dtype=np.int64)
        sign = 1 - 2 * par
        total += term.coeff * (1j ** ny) * np.sum(sign * np.conj(psi[idx ^ x]) * psi)
    return total


# ------------------------------------------------------------------ commands

def cmd_schedule(cfg, out):
    """cmd_schedule, report.cpp:114-147."""
    circuit, shape = _load_circuit(cfg, False)
    shape = _resolve_shape(cfg, shape)
    deps = qb.build_dependency_graph(circuit)
    names = [cfg.scheduler] + [s for s in cfg.compare if s != cfg.scheduler]
    report = {"config": _config_echo(cfg, shape)}
    results = {}
    for name in names:
        t0 = time.perf_counter()
        s = _scheduler(name, circuit, deps, shape)
        ms = (time.perf_counter() - t0) * 1e3
        results[name] = {"metrics": _metrics(s, cfg.w, ms), "schedule": json.loads(qb.schedule_to_json(s))}
    if len(names) == 1:
        report.update(results[names[0]])
    else:
        report["results"] = results
    _emit(cfg, out, _dumps(report))
    return 0


def cmd_simulate(cfg, out, diag):
    """cmd_simulate, report.cpp:149-192, on the B200 backend."""
    circuit, shape = _load_circuit(cfg, True)
    shape = _resolve_shape(cfg, shape)
    for op in circuit.operators:
        if op.is_gate and op.payload is None:
            raise qb.MissingPayload(f"gate {op.id} has no payload")
    qb.init_distributed()
    deps = qb.build_dependency_graph(circuit)
    sched = _scheduler(cfg.scheduler, circuit, deps, shape)
    st = qb.init_state(circuit.n, shape)
    qb.run_qsu(st, circuit, sched, cfg.workers)
    final = qb.flatten(st)
    report = {"config": _config_echo(cfg, shape), "n": circuit.n, "norm": st.norm(), "qr_executed": len(st.qr_log),
              "relocated_total": st.total_relocated}
    code = 0
    if cfg.verify:
        if circuit.n > qb.kOracleMaxQubits:
            raise qb.OracleTooLarge(f"--verify needs n <= {qb.kOracleMaxQubits}")
        psi = np.zeros(1 << circuit.n, dtype=complex)
        psi[0] = 1
        for op in circuit.operators:
            psi = _dense_apply(psi, circuit.n, op)
        worst = float(np.max(np.abs(psi - final)))
        ok = worst <= 1e-12
        report["verify"] = {"max_amp_error": worst, "pass": ok}
        code = 0 if ok else 1
    if cfg.out:
        try:
            with open(cfg.out, "wb") as f:
                f.write(qb.write_state_dump(final, shape.p))
        except OSError:  # report.cpp:184-185: ConfigError, exit code 2
            raise qb.ConfigError(f"cannot write output file: {cfg.out}") from None
        report["dump"] = cfg.out
    out.write(_dumps(report))
    if code:
        diag.write("verification failed\n")
    return code


def cmd_evc(cfg, out, diag):
    """cmd_evc, report.cpp:194-259, on the B200 backend."""
    terms, n = _load_hamiltonian(cfg)
    circuit = None
    if cfg.circuit:
        try:
            circuit = qb.seed_payloads(parse_circuit(open(cfg.circuit).read()), cfg.seed)
        except OSError:
            raise qb.ConfigError(f"cannot open circuit file: {cfg.circuit}") from None
        if circuit.n != n:
            raise qb.ConfigError(f"circuit has {circuit.n} qubits, Hamiltonian has {n}")
    shape = _resolve_shape(cfg, qb.ClusterShape.flat(1))
    qb.init_distributed()
    st = qb.init_state(n, shape)
    if circuit is not None:
        sched = _scheduler(cfg.scheduler, circuit, qb.build_dependency_graph(circuit), shape)
        qb.run_qsu(st, circuit, sched, cfg.workers)
    t0 = time.perf_counter()
    plan = qb.plan_evc(terms, n, shape, cfg.diagonalize != "off", cfg.workers)
    ms = (time.perf_counter() - t0) * 1e3
    energy = qb.expectation(st, plan, terms, cfg.workers)
    base = qb.index_order_baseline(terms, n, shape)
    report = {"config": _config_echo(cfg, shape), "n": n, "terms": len(terms), "energy": energy.real,
              "energy_imag": energy.imag, "tiles": len(plan.tiles), "n_qr": plan.qr_count(),
              "baseline_qr": base.n_qr, "ratio": base.n_qr / max(1, plan.qr_count()), "sched_time_ms": ms,
              "plan": json.loads(qb.plan_to_json(plan))}
    code = 0
    if cfg.verify:
        if n > qb.kOracleMaxQubits:
            raise qb.OracleTooLarge(f"--verify needs n <= {qb.kOracleMaxQubits}")
        psi = np.zeros(1 << n, dtype=complex)
        psi[0] = 1
        if circuit is not None:
            for op in circuit.operators:
                psi = _dense_apply(psi, n, op)
        dense = _dense_expectation(psi, n, terms)
        err = abs(energy - dense)
        ok = err <= 1e-10 * (1 + abs(dense)) and abs(energy.imag) <= 1e-10
        report["verify"] = {"dense_energy": dense.real, "abs_error": err, "pass": ok}
        code = 0 if ok else 1
    _emit(cfg, out, _dumps(report))
    if code:
        diag.write("verification failed\n")
    return code


def cmd_bench(cfg, out):
    """cmd_bench, report.cpp:261-280: scheduler sweep over GateFabric (CSV)."""
    buf = io.StringIO()
    buf.write("n,p,scheduler,n_qr,n_intra,n_inter,cost,sched_time_ms\n")
    shape = _resolve_shape(cfg, qb.ClusterShape.flat(4))
    for n in cfg.sweep_n:
        circuit = qb.gen_gatefabric(n, cfg.layers, cfg.seed, False)
        deps = qb.build_dependency_graph(circuit)
        for name in cfg.schedulers:
            t0 = time.perf_counter()
            s = _scheduler(name, circuit, deps, shape)
            ms = (time.perf_counter() - t0) * 1e3
            c = qb.count_qrs(s)
            buf.write(f"{n},{shape.p},{name},{c.total},{c.intra},{c.inter},{qb.qr_cost(c, cfg.w):g},{ms:g}\n")
    _emit(cfg, out, buf.getvalue())
    return 0


# ------------------------------------------------------------------ main

def _parser():
    ap = argparse.ArgumentParser(prog="qrtile", description="Lazy qubit-reordering scheduler and B200 simulator")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--fixture", default="")
        p.add_argument("--circuit", default="")
        p.add_argument("--hamiltonian", default="")
        p.add_argument("--p", type=int, default=0)
        p.add_argument("--nodes", type=int, default=0)
        p.add_argument("--gpn", type=int, default=0)
        p.add_argument("--scheduler", default="flat", choices=SCHEDULERS)
        p.add_argument("--weights", default="")
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--workers", type=int, default=1)
        p.add_argument("--out", default="")
        p.add_argument("--format", default="json", choices=("json", "csv"))
        p.add_argument("--config", default="")

    p = sub.add_parser("schedule")
    common(p)
    p.add_argument("--compare", default="")
    p = sub.add_parser("simulate")
    common(p)
    p.add_argument("--verify", action="store_true")
    p = sub.add_parser("evc")
    common(p)
    p.add_argument("--diagonalize", default="on", choices=("on", "off"))
    p.add_argument("--verify", action="store_true")
    p = sub.add_parser("bench")
    common(p)
    p.add_argument("--sweep-n", default="")
    p.add_argument("--layers", type=int, default=2)
    p.add_argument("--schedulers", default="flat,hierarchical,adhoc")
    return ap


def _with_config_file(ap, argv):
    """--config key=value file; command-line flags win."""
    args = ap.parse_args(argv)
    if not args.config:
        return args
    try:
        lines = open(args.config).read().splitlines()
    except OSError:
        raise qb.ConfigError(f"cannot open config file: {args.config}") from None
    given = {a.split("=", 1)[0] for a in argv if a.startswith("--")}
    extra = []
    for line in lines:
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise qb.ConfigError(f"config line without '=': {line}")
        key, val = (s.strip() for s in line.split("=", 1))
        flag = "--" + key
        if flag in given:
            continue
        if val.lower() in ("true", "false"):
            if val.lower() == "true":
                extra.append(flag)
        else:
            extra += [flag, val]
    return ap.parse_args([argv[0]] + extra + argv[1:])


def main(argv=None, out=None, diag=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    out = out or sys.stdout
    diag = diag or sys.stderr
    ap = _parser()
    try:
        cfg = _with_config_file(ap, argv)
    except SystemExit as e:  # argparse usage error
        return 2 if e.code else 0
    except qb.Error as e:
        diag.write(f"error: {e}\n")
        return 2
    try:
        cfg.w = _weights(cfg.weights)
        split = [s for s in getattr(cfg, "compare", "").split(",") if s]
        cfg.compare = split
        if cfg.cmd == "bench":
            cfg.sweep_n = [int(x) for x in cfg.sweep_n.split(",") if x]
            cfg.schedulers = [s for s in cfg.schedulers.split(",") if s]
        if not hasattr(cfg, "diagonalize"):
            cfg.diagonalize = "on"
        if not hasattr(cfg, "verify"):
            cfg.verify = False
        if cfg.workers < 1:
            raise qb.ConfigError("--workers must be at least 1")
        if cfg.cmd == "schedule":
            return cmd_schedule(cfg, out)
        if cfg.cmd == "simulate":
            return cmd_simulate(cfg, out, diag)
        if cfg.cmd == "evc":
            return cmd_evc(cfg, out, diag)
        return cmd_bench(cfg, out)
    except (qb.Error, ValueError) as e:
        diag.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
