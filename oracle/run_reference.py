"""TEST INFRASTRUCTURE ONLY: run the real reference solver on a named synthetic
instance and record a golden JSON (status, counts, objective, residuals, the
per-check progress trace, versions and host info).

    python oracle/run_reference.py <instance-spec> <out.json> [--eps 1e-8] [--time-limit S]
                                   [--iter-limit N] [--theta T] [--eta-scale E]

The golden also counts the calls of the reference's two rollback branches
(``rollbacks``: overflow halt / divergence), found from the calling source.

Instance specs are resolved by ``oracle/instances.py`` so the GPU tests build
the identical instance from the same spec string.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import scipy  # noqa: E402

import instances  # noqa: E402
import refbridge  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("spec")
    ap.add_argument("out")
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--time-limit", type=float, default=None)
    ap.add_argument("--iter-limit", type=int, default=1_000_000)
    ap.add_argument("--theta", type=float, default=None)
    ap.add_argument("--eta-scale", type=float, default=None)
    args = ap.parse_args(argv)
    aq = refbridge.load_reference()
    assert aq is not None and aq.active_backend() == "cython"
    # count the two rollback branches of the reference loop (engine.py:407-417
    # overflow halt, engine.py:484-487 divergence) by the calling line
    import inspect

    from anchorqp import engine as ref_engine

    rollbacks = {"overflow": 0, "divergence": 0}
    orig = ref_engine._rollback_round

    def counted(state):
        src = inspect.getsource(inspect.currentframe().f_back).splitlines()
        line = inspect.currentframe().f_back.f_lineno - inspect.getsourcelines(inspect.currentframe().f_back)[1]
        ctx = "\n".join(src[max(0, line - 6):line + 1])
        rollbacks["overflow" if "isfinite(move)" in ctx else "divergence"] += 1
        return orig(state)

    ref_engine._rollback_round = counted
    t0 = time.time()
    ours = instances.build(args.spec)
    if args.spec.startswith("qps:"):  # the reference's own reader on the same file
        with open(args.spec.split(":", 1)[1]) as f:
            prob = aq.parse_qps(f.read()).problem
    else:
        prob = refbridge.to_reference(ours, aq)
    gen_s = time.time() - t0
    trace = []

    def progress(it, rep, omega, rnd):
        trace.append([it, rep.r_primal, rep.r_dual, rep.r_gap, omega, rnd])

    extra = {}
    if args.theta is not None:
        extra["theta"] = args.theta
    if args.eta_scale is not None:
        extra["eta_scale"] = args.eta_scale
    params = aq.SolverParams(eps_tol=args.eps, time_limit=args.time_limit, iter_limit=args.iter_limit, **extra)
    res = aq.solve(prob, params, progress=progress)
    rep = res.report
    out = dict(
        spec=args.spec, eps_tol=args.eps, time_limit=args.time_limit, iter_limit=args.iter_limit,
        status=res.status.value, outer=res.outer_iterations, inner=res.inner_iterations,
        restarts=res.restarts, seconds=res.seconds, gen_seconds=gen_s,
        objective=rep.primal_objective, dual_objective=rep.dual_objective,
        r_primal=rep.r_primal, r_dual=rep.r_dual, r_gap=rep.r_gap, kkt=rep.kkt_max,
        certificate=None if res.certificate is None else dict(
            kind=res.certificate.kind.value, violation=res.certificate.violation,
            improvement=res.certificate.improvement),
        x_norm=float(np.linalg.norm(res.x)), y_norm=float(np.linalg.norm(res.y)),
        n=ours.n, m=ours.m, trace=trace, params=extra, rollbacks=rollbacks,
        versions=dict(numpy=np.__version__, scipy=scipy.__version__, python=platform.python_version(),
                      anchorqp=aq.__version__, backend=aq.active_backend()),
        host=dict(cpu=platform.processor() or platform.machine(), nproc=os.cpu_count(),
                  openblas_threads=os.environ.get("OPENBLAS_NUM_THREADS")),
    )
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("spec", "status", "outer", "inner", "restarts", "seconds", "objective", "kkt",
                                          "rollbacks")}))


if __name__ == "__main__":
    main()
