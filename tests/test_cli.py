"""CPU: the command line (paper_2602_23967_b200/cli.py) against the reference's
(aq/cli.py): usage / parse exit codes and the `gen` files, byte for byte.
The solving commands are in tests/test_gpu_cli.py."""

import pytest

import refbridge
from paper_2602_23967_b200 import random_qp
from paper_2602_23967_b200.cli import EXIT_PARSE, EXIT_USAGE, TRACE_HEADER, main
from paper_2602_23967_b200.io import write_qps

AQ = refbridge.load_reference()
needs_ref = pytest.mark.skipif(AQ is None, reason="oracle/_ref not built")


@pytest.fixture
def toy(tmp_path):
    path = tmp_path / "toy.qps"
    path.write_text(write_qps(random_qp(5, 3, "diagonal", seed=1)))
    return str(path)


@pytest.mark.parametrize("argv", [
    ["solve", "--input", "{toy}", "--tol", "0"],
    ["solve", "--input", "{toy}", "--inf-tol", "-1"],
    ["solve", "--input", "{toy}", "--pid", "1,2"],
    ["solve", "--input", "{toy}", "--pid", "a,b,c"],
    ["solve", "--input", "{toy}", "--frobnicate"],
    ["solve", "--input", "{toy}", "--theta", "1.5"],
    ["frobnicate"],
    ["bench", "--dir", "{empty}"],
])
def test_usage_errors_exit_64(toy, tmp_path, argv):
    (tmp_path / "empty").mkdir()
    argv = [a.format(toy=toy, empty=str(tmp_path / "empty")) for a in argv]
    assert main(argv) == EXIT_USAGE


def test_input_and_parse_errors_exit_65(tmp_path):
    assert main(["solve", "--input", "/nonexistent.qps"]) == EXIT_PARSE
    bad = tmp_path / "bad.qps"
    bad.write_text("COLUMNS\n x obj 1.0\n")
    assert main(["solve", "--input", str(bad)]) == EXIT_PARSE


def test_trace_header_is_the_reference_header():
    assert TRACE_HEADER == "iteration,r_primal,r_dual,r_gap,omega,round"


@needs_ref
@pytest.mark.parametrize("argv", [
    ["gen", "--kind", "random", "--n", "6", "--m", "3", "--seed", "2"],
    ["gen", "--kind", "random", "--n", "40", "--m", "25", "--structure", "diagonal", "--density", "0.2"],
    ["gen", "--kind", "lasso", "--n", "5", "--m", "12", "--format", "json"],
    ["gen", "--kind", "random", "--n", "30", "--m", "10", "--structure", "low_rank", "--format", "json"],
])
def test_gen_files_equal_the_reference_cli(tmp_path, argv):
    from anchorqp.cli import cli_main as ref_main

    ext = ".json" if "json" in argv else ".qps"
    ours, theirs = tmp_path / f"ours{ext}", tmp_path / f"ref{ext}"
    assert main(argv + ["--output", str(ours)]) == 0
    assert ref_main(argv + ["--output", str(theirs)]) == 0
    assert ours.read_text() == theirs.read_text()
