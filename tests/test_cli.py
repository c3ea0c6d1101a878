"""The `qrtile`-compatible command-line driver (paper_2410_04252_b200/cli.py),
mirroring the reference's CLI integration tests (proj/tests/test_cli.cpp:45-217):
report keys, golden counts, exit codes, config-file precedence, state dumps.
`schedule` / `bench` are host-only; `simulate` / `evc` run on the B200."""
import io
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def run(args, tmp=None):
    from paper_2410_04252_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    code = cli.main(args.split(), out, err)
    return code, out.getvalue(), err.getvalue()


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


# ------------------------------------------------------------- host-only

def test_schedule_gatefabric_counts():  # test_cli.cpp:45-57
    code, out, _ = run("schedule --fixture gatefabric-fig6 --p 16 --scheduler flat")
    assert code == 0
    r = json.loads(out)
    assert r["metrics"]["n_qr"] == 3 and len(r["schedule"]["tiles"][0]["gates"]) == 9
    code, out, _ = run("schedule --fixture gatefabric-fig6 --nodes 4 --gpn 4 --scheduler hierarchical")
    r = json.loads(out)
    assert code == 0 and r["metrics"]["n_inter"] == 2 and r["metrics"]["n_intra"] == 3


def test_schedule_all_local_zero_qrs(tmp_path):  # :59-69
    path = write(tmp_path, "all_local.qct", "n 6\nG 0 0 1\nG 1 2\nG 2 1 2\n")
    code, out, _ = run(f"schedule --circuit {path} --p 4 --scheduler adhoc")
    assert code == 0 and json.loads(out)["metrics"]["n_qr"] == 0


def test_schedule_compare():  # :71-86
    code, out, _ = run("schedule --fixture gatefabric-fig6 --nodes 4 --gpn 4 --scheduler flat "
                       "--compare adhoc,hierarchical --weights 1,24")
    assert code == 0
    res = json.loads(out)["results"]
    assert res["flat"]["metrics"]["cost"] == pytest.approx(72.0)
    assert res["hierarchical"]["metrics"]["cost"] == pytest.approx(51.0)
    assert res["flat"]["metrics"]["n_qr"] <= res["adhoc"]["metrics"]["n_qr"]


def test_bench_csv_rows():  # :168-192
    code, out, _ = run("bench --sweep-n 8,12,16 --p 4 --layers 2 --schedulers flat,adhoc")
    assert code == 0
    lines = [l for l in out.splitlines() if l]
    assert lines[0] == "n,p,scheduler,n_qr,n_intra,n_inter,cost,sched_time_ms"
    rows = lines[1:]
    assert len(rows) == 6
    for i in range(0, 6, 2):
        assert int(rows[i].split(",")[3]) <= int(rows[i + 1].split(",")[3])


def test_bench_empty_sweep():  # :194-198
    code, out, _ = run("bench --p 4")
    assert code == 0 and out == "n,p,scheduler,n_qr,n_intra,n_inter,cost,sched_time_ms\n"


def test_config_violations_exit_2():  # :200-205 (the evc case needs a device: see the GPU test)
    assert run("schedule --fixture gatefabric-fig6 --p 3")[0] == 2
    assert run("schedule --p 4")[0] == 2
    assert run("schedule --fixture nope --p 4")[0] == 2
    assert run("schedule --fixture gatefabric-fig6 --bogus")[0] == 2


def test_reports_reproducible():  # :207-217 (timings excluded)
    args = "schedule --fixture gatefabric-fig6 --nodes 4 --gpn 4 --scheduler hierarchical"
    a, b = json.loads(run(args)[1]), json.loads(run(args)[1])
    for r in (a, b):
        r["metrics"].pop("sched_time_ms")
    assert a == b


def test_config_file_overridden_by_flags(tmp_path):  # :219-226
    cfg = write(tmp_path, "conf.ini", "p=8\nscheduler=adhoc\n")
    code, out, _ = run(f"schedule --fixture gatefabric-fig6 --config {cfg} --p 16")
    r = json.loads(out)
    assert code == 0 and r["config"]["p"] == 16 and r["config"]["scheduler"] == "adhoc"


def test_text_formats_round_trip(qb):
    from paper_2410_04252_b200 import cli

    c = qb.gen_random_circuit(9, 50, 11, 3, False)
    c2 = cli.parse_circuit(cli.serialize_circuit(c))
    assert c2.n == c.n and [list(o.targets) for o in c2.operators] == [list(o.targets) for o in c.operators]
    terms = qb.gen_synthetic_jw(8, 3)
    t2, n = cli.parse_hamiltonian(cli.serialize_hamiltonian(terms, 8))
    assert n == 8 and [t.letters for t in t2] == [t.letters for t in terms]
    assert [t.coeff for t in t2] == [t.coeff for t in terms]  # %.17g round trip is exact
    with pytest.raises(qb.ParseError):
        cli.parse_circuit("n 3\nG 1 0\n")  # ids must be dense
    with pytest.raises(qb.IndexError):
        cli.parse_hamiltonian("n 2\n1 0 Z5\n")


def test_module_entry_point():
    res = subprocess.run([sys.executable, "-m", "paper_2410_04252_b200.cli", "schedule", "--p", "4"], cwd=ROOT,
                         capture_output=True, text=True, timeout=120)
    assert res.returncode == 2 and "no circuit input" in res.stderr


# ------------------------------------------------------------- on the B200

@pytest.mark.gpu
def test_simulate_verify_random_circuit(qb, device, tmp_path):  # :88-97
    from paper_2410_04252_b200 import cli

    path = write(tmp_path, "rand.qct", cli.serialize_circuit(qb.gen_random_circuit(10, 40, 2024, 2, False)))
    code, out, _ = run(f"simulate --circuit {path} --p 4 --verify --seed 7")
    r = json.loads(out)
    assert code == 0 and r["verify"]["pass"] and r["verify"]["max_amp_error"] <= 1e-12


@pytest.mark.gpu
def test_simulate_dumps_identical_across_p(qb, device, tmp_path):  # :99-118
    from paper_2410_04252_b200 import cli

    path = write(tmp_path, "dump.qct", cli.serialize_circuit(qb.gen_random_circuit(8, 30, 99, 2, False)))
    d1, d8 = str(tmp_path / "p1.bin"), str(tmp_path / "p8.bin")
    assert run(f"simulate --circuit {path} --p 1 --seed 5 --out {d1}")[0] == 0
    assert run(f"simulate --circuit {path} --p 8 --seed 5 --out {d8}")[0] == 0
    a1, _, p1 = qb.read_state_dump(open(d1, "rb").read())
    a8, _, p8 = qb.read_state_dump(open(d8, "rb").read())
    assert p1 == 1 and p8 == 8 and float(np.max(np.abs(a1 - a8))) <= 1e-12


@pytest.mark.gpu
def test_empty_circuit_dump_is_zero_state(qb, device, tmp_path):  # :120-129
    path = write(tmp_path, "empty.qct", "n 4\n")
    dump = str(tmp_path / "empty.bin")
    assert run(f"simulate --circuit {path} --p 2 --out {dump}")[0] == 0
    amps, n, _ = qb.read_state_dump(open(dump, "rb").read())
    assert amps[0] == 1.0 and np.all(amps[1:] == 0)


@pytest.mark.gpu
def test_evc_z0_and_jw12(qb, device, tmp_path):  # :131-151
    path = write(tmp_path, "z0.ham", "n 4\n1 0 Z0\n")
    code, out, _ = run(f"evc --hamiltonian {path} --p 2 --verify")
    r = json.loads(out)
    assert code == 0 and r["energy"] == pytest.approx(1.0) and r["verify"]["pass"]
    code, out, _ = run("evc --fixture jw12 --p 4 --verify")
    r = json.loads(out)
    assert code == 0 and r["n_qr"] <= 5 and r["ratio"] >= 20.0 and r["verify"]["pass"]
    assert run("evc --fixture jw12 --p 4 --diagonalize off")[0] == 2  # too wide (:204)


@pytest.mark.gpu
def test_evc_diagonalize_tiles_and_circuit(qb, device, tmp_path):  # :153-166 + a circuit before EVC
    from paper_2410_04252_b200 import cli

    path = write(tmp_path, "small.ham", "n 6\n1 0 X0 X1\n0.5 0 Z2 Z3\n0.25 0 X4 X5\n")
    on = json.loads(run(f"evc --hamiltonian {path} --p 4 --diagonalize on")[1])
    off = json.loads(run(f"evc --hamiltonian {path} --p 4 --diagonalize off")[1])
    assert on["tiles"] <= off["tiles"]
    ham = write(tmp_path, "jw8.ham", cli.serialize_hamiltonian(qb.gen_synthetic_jw(8, 2), 8))
    circ = write(tmp_path, "gf8.qct", cli.serialize_circuit(qb.gen_gatefabric(8, 6, 1, False)))
    code, out, _ = run(f"evc --hamiltonian {ham} --circuit {circ} --p 2 --verify --seed 3")
    assert code == 0 and json.loads(out)["verify"]["pass"]


@pytest.mark.gpu
def test_simulate_unwritable_dump_exit_2(qb, device, tmp_path):  # report.cpp:184-185
    path = write(tmp_path, "empty.qct", "n 4\n")
    code, _, err = run(f"simulate --circuit {path} --p 2 --out {tmp_path}/no/such/dir/x.bin")
    assert code == 2 and "cannot write output file" in err
