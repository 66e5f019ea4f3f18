"""GPU: the reference's OWN test suite (anchorqp/tests, copied into the
git-ignored oracle/_ref/tests by oracle/build_ref.sh) run against this build
through the drop-in boundaries -- anchorqp.solve routed to the B200 solve and
the B200 kernels registered as reference backend "cuda"
(oracle/ref_suite_plugin.py).

One reference test cannot pass with ANY CUDA backend and is expected to fail:
test_bench.py::TestHarness::test_parallel_matches_serial runs solves in a
fork()ed process pool (aq/bench.py:94-97), and CUDA cannot be initialised in a
forked child; batch.solve_many (streams) replaces that pool on a GPU."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
SUITE = os.path.join(ROOT, "oracle", "_ref", "tests")
EXPECTED_FAIL = {"oracle/_ref/tests/test_bench.py::TestHarness::test_parallel_matches_serial"}


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="oracle/_ref/tests missing (run oracle/build_ref.sh)")
def test_reference_suite_passes_on_b200(cuda):
    report = os.path.join(ROOT, "build", "ref_suite_report.json")
    os.makedirs(os.path.dirname(report), exist_ok=True)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "oracle", "_ref"),
                                                       os.path.join(ROOT, "oracle"), ROOT]),
               AQP_REF_SUITE_REPORT=report)
    out = subprocess.run([sys.executable, "-m", "pytest", "oracle/_ref/tests", "-p", "ref_suite_plugin", "-q",
                          "-rf", "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=1200)
    failed = {line.split()[1] for line in out.stdout.splitlines() if line.startswith("FAILED ")}
    summary = out.stdout.strip().splitlines()[-1]
    assert failed <= EXPECTED_FAIL, f"{summary}\n{out.stdout[-4000:]}"
    assert " passed" in summary and "error" not in summary, summary
    # how many of the passing tests actually exercise the B200 build (the rest
    # test the reference's own Python: model, QPS, certify internals ...)
    import json

    rep = json.load(open(report))
    print({k: v for k, v in rep.items() if k != "records"})
    assert rep["passed_via_b200_solve"] >= 20 and rep["passed_touching_b200"] >= 60
