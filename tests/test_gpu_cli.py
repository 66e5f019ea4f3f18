"""GPU: the command line's solving subcommands (cli.py) -- the reference CLI
tests' cases (aq tests/test_cli.py) plus parity of the result document with
the reference CLI run on the same file."""

import json

import numpy as np
import pytest

import refbridge
from paper_2602_23967_b200 import random_qp
from paper_2602_23967_b200.cli import TRACE_HEADER, main
from paper_2602_23967_b200.io import dump_problem_json, write_qps

pytestmark = pytest.mark.gpu
AQ = refbridge.load_reference()


@pytest.fixture
def toy(tmp_path):
    path = tmp_path / "toy.qps"
    path.write_text(write_qps(random_qp(5, 3, "diagonal", seed=1)))
    return str(path)


def test_optimal_exit_document_and_trace(cuda, toy, tmp_path):
    out, trace = tmp_path / "r.json", tmp_path / "t.csv"
    assert main(["solve", "--input", toy, "--tol", "1e-6", "--output", str(out), "--trace", str(trace)]) == 0
    doc = json.loads(out.read_text())
    assert doc["status"] == "optimal" and doc["instance"] == "toy.qps"
    for key in ("primal_objective", "dual_objective", "r_primal", "r_dual", "r_gap", "outer_iterations",
                "inner_iterations", "restarts", "seconds"):
        assert key in doc
    lines = trace.read_text().strip().splitlines()
    assert lines[0] == TRACE_HEADER and len(lines) >= 2
    for line in lines[1:]:
        f = line.split(",")
        assert len(f) == 6
        int(f[0]), float(f[1]), int(f[5])


@pytest.mark.parametrize("text,code,status", [
    ("ROWS\n N obj\n L c1\nCOLUMNS\n x obj 0.0 c1 1.0\nRHS\n RHS c1 -1.0\nENDATA\n", 2, "primal_infeasible"),
    ("ROWS\n N obj\nCOLUMNS\n x obj -1.0\nENDATA\n", 3, "dual_infeasible"),
])
def test_infeasibility_exit_codes(cuda, tmp_path, text, code, status):
    path = tmp_path / "p.qps"
    path.write_text(text)
    out = tmp_path / "r.json"
    assert main(["solve", "--input", str(path), "--output", str(out)]) == code
    doc = json.loads(out.read_text())
    assert doc["status"] == status and "certificate" in doc


def test_iteration_limit_exit_code(cuda, toy):
    assert main(["solve", "--input", toy, "--tol", "1e-12", "--iter-limit", "5"]) == 4


def test_bench_directory(cuda, tmp_path, capsys):
    for seed in range(2):
        (tmp_path / f"i{seed}.qps").write_text(write_qps(random_qp(4, 2, "diagonal", seed=seed)))
    dump_problem_json(random_qp(4, 2, "sparse", seed=5), tmp_path / "i2.json")
    out = tmp_path / "summary.json"
    assert main(["bench", "--dir", str(tmp_path), "--tol", "1e-6", "--time-limit", "100", "--output", str(out),
                 "--streams", "3"]) == 0
    assert "SGM10" in capsys.readouterr().out
    doc = json.loads(out.read_text())
    assert doc["summary"]["instances"] == 3 and len(doc["records"]) == 3


@pytest.mark.skipif(AQ is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("fname", ["qps_mixed_400.qps"])
def test_result_document_matches_reference_cli(cuda, tmp_path, fname):
    """Same file, same flags: our `solve` and the reference's produce the same
    status, the same first trace rows (iteration and round columns), and
    outer counts / objectives within the north-star contract."""
    import os

    from anchorqp.cli import cli_main as ref_main

    path = os.path.join(os.path.dirname(__file__), "golden", fname)
    flags = ["--tol", "1e-8"]
    ours, theirs = tmp_path / "o.json", tmp_path / "r.json"
    tro, trr = tmp_path / "o.csv", tmp_path / "r.csv"
    assert main(["solve", "--input", path, "--output", str(ours), "--trace", str(tro)] + flags) == 0
    assert ref_main(["solve", "--input", path, "--output", str(theirs), "--trace", str(trr)] + flags) == 0
    a, b = json.loads(ours.read_text()), json.loads(theirs.read_text())
    assert a["status"] == b["status"] and a["instance"] == b["instance"]
    assert abs(a["outer_iterations"] - b["outer_iterations"]) <= 0.10 * b["outer_iterations"]
    assert abs(a["primal_objective"] - b["primal_objective"]) <= 1e-6 * max(1.0, abs(b["primal_objective"]))
    rows = lambda p: [tuple(int(l.split(",")[i]) for i in (0, 5)) for l in p.read_text().splitlines()[1:]]
    ro, rr = rows(tro), rows(trr)
    assert ro[:5] == rr[:5]  # the same certification points and rounds early on
