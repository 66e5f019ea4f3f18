"""TEST INFRASTRUCTURE ONLY: a pytest plugin that runs the reference's OWN
test suite (copied by oracle/build_ref.sh into oracle/_ref/tests, git-ignored)
against this repo, through the two drop-in boundaries of INTEGRATION.md:

* the kernel registry: this package's ``kernels`` module is registered as the
  reference backend "cuda" (``anchorqp/_kernels/__init__.py:29``) and selected as
  the active backend, so every reference function that calls a kernel runs on
  the B200 kernels, and every ``kernel_backend``-parametrised test also runs them;
* the solve entry point: ``anchorqp.solve`` / ``anchorqp.engine.solve`` are
  routed to ``paper_2602_23967_b200.solve`` and its result is rebuilt as the
  reference's own ``SolveResult`` / ``ResidualReport`` / ``Certificate``.

    PYTHONPATH=oracle/_ref:oracle:. python -m pytest oracle/_ref/tests -p ref_suite_plugin
"""

import json
import os

import anchorqp
import anchorqp.certify as rcert
import anchorqp.engine as reng
import anchorqp.errors as rerr
from anchorqp import _kernels as rkern

import paper_2602_23967_b200 as b200
from paper_2602_23967_b200 import errors as b200_errors
from paper_2602_23967_b200 import kernels as b200_kernels

# which tests actually reach the B200 path (AQP_REF_SUITE_REPORT=<path>: a
# per-session JSON summary): a test "reaches" it when it calls the routed
# solve or a kernel of the "cuda" backend
_hits = {"solve": False, "kernel": False}
_records = []


class _CountingBackend:
    """The B200 kernel module as seen by the reference registry, counting calls."""

    def __init__(self, mod):
        self._mod = mod

    def __getattr__(self, name):
        f = getattr(self._mod, name)
        if not callable(f):
            return f

        def counted(*a, **k):
            _hits["kernel"] = True
            return f(*a, **k)

        return counted


rkern._BACKENDS["cuda"] = _CountingBackend(b200_kernels)
_reference_solve = reng.solve
# the B200 kernels are the ACTIVE backend for the whole suite (the reference's
# own Python -- pdhg_step, solve_bb, residuals, linalg products -- then runs on
# them wherever it calls a kernel); AQP_REF_SUITE_BACKEND=cython keeps the
# reference's default and only routes the kernel_backend-parametrised tests
rkern.select_backend(os.environ.get("AQP_REF_SUITE_BACKEND", "cuda"))


def _to_reference(res):
    rep = res.report
    report = rcert.ResidualReport(r_primal=rep.r_primal, r_dual=rep.r_dual, r_gap=rep.r_gap,
                                  primal_objective=rep.primal_objective, dual_objective=rep.dual_objective,
                                  dual_slack=rep.dual_slack)
    cert = None
    if res.certificate is not None:
        c = res.certificate
        cert = rcert.Certificate(kind=rcert.CertificateKind(c.kind.value), ray=c.ray, violation=c.violation,
                                 improvement=c.improvement)
    return reng.SolveResult(status=reng.SolveStatus(res.status.value), x=res.x, y=res.y, report=report,
                            certificate=cert, outer_iterations=res.outer_iterations,
                            inner_iterations=res.inner_iterations, restarts=res.restarts, seconds=res.seconds)


def _reraise_as_reference(exc):
    """Our error classes mirror the reference's names (aq/errors.py); raise the
    reference's class so ``pytest.raises(anchorqp.errors.X)`` sees it."""
    cls = getattr(rerr, type(exc).__name__, None)
    if isinstance(cls, type) and issubclass(cls, BaseException):
        raise cls(str(exc)) from exc
    raise exc


def b200_solve(problem, params=None, progress=None):
    """anchorqp.solve's signature, executed on the B200 path."""
    cb = None
    if progress is not None:
        def cb(k, rep, omega, rnd):
            progress(k, rcert.ResidualReport(r_primal=rep.r_primal, r_dual=rep.r_dual, r_gap=rep.r_gap,
                                             primal_objective=rep.primal_objective,
                                             dual_objective=rep.dual_objective, dual_slack=rep.dual_slack),
                     omega, rnd)
    _hits["solve"] = True
    try:
        res = b200.solve(problem, params, cb)
    except b200_errors.SolverError as exc:
        _reraise_as_reference(exc)
    return _to_reference(res)


anchorqp.solve = b200_solve
reng.solve = b200_solve


def pytest_report_header(config):
    return ["reference suite routed to the B200 build: anchorqp.solve -> paper_2602_23967_b200.solve, "
            "kernel backend 'cuda' -> paper_2602_23967_b200.kernels"]


def pytest_runtest_setup(item):
    _hits["solve"] = _hits["kernel"] = False


def pytest_runtest_logreport(report):
    if report.when == "call":
        _records.append({"test": report.nodeid, "outcome": report.outcome, "solve": _hits["solve"],
                         "kernel": _hits["kernel"]})


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("AQP_REF_SUITE_REPORT")
    if not path:
        return
    passed = [r for r in _records if r["outcome"] == "passed"]
    summary = {
        "tests": len(_records), "passed": len(passed),
        "passed_via_b200_solve": sum(r["solve"] for r in passed),
        "passed_via_b200_kernels_only": sum(r["kernel"] and not r["solve"] for r in passed),
        "passed_touching_b200": sum(r["solve"] or r["kernel"] for r in passed),
        "passed_reference_python_only": sum(not (r["solve"] or r["kernel"]) for r in passed),
        "records": _records,
    }
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
