"""TEST INFRASTRUCTURE ONLY: time the reference CPU solver on a bounded
sample of a workload, for bench.py's ``cpu_baseline`` and ``--impl reference``.

The reference runs unmodified through its public ``anchorqp.solve``; the
only instrumentation is a pass-through wrapper around
``anchorqp.engine.pdhg_step`` (called once per outer iteration,
aq/engine.py:397) that records its start time and the BB inner iterations it
returns.  A sample of K outer iterations after W warm-up iterations is timed
from the start of step W to the start of step W+K, i.e. it covers every
per-iteration cost (A'y, the BB solve, A xbar, Halpern, norms, window sums).
The GPU arm of bench.py times the same outer iterations [W, W+K) of the same
solve (engine.solve's ``marks``).

Initialisation is outside the timed range.  Its power iteration
(``estimate_norm``, 100 x A'A) is served from ``oracle/norm_memo.py``'s
recordings of the reference's own result on the bench instances when the
matrix fingerprint matches (a bitwise-identical float, so the trajectory is
unchanged) -- on C5 that saves ~6 minutes of single-core work per run.

When the built reference (oracle/_ref) is absent the oracle port
(oracle/oracle.py, bit-identical trajectory) is timed instead.

    python oracle/ref_bench.py <spec> <warmup> <steps>   -> one JSON line
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def run_problem(problem, warmup: int, steps: int, eps: float = 1e-8, spec: str = ""):
    import refbridge

    aq = refbridge.load_reference()
    starts, inners = [], []
    if aq is None:
        return _run_port(problem, warmup, steps, eps, spec)
    import anchorqp.engine as eng
    import norm_memo

    inner_step = eng.pdhg_step
    orig_norm = eng.estimate_norm
    norm_memo.patch(aq)

    def timed_step(*a, **k):
        starts.append(time.perf_counter())
        out = inner_step(*a, **k)
        inners.append(out[1])
        return out

    eng.pdhg_step = timed_step
    try:
        t0 = time.perf_counter()
        ref_problem = refbridge.to_reference(problem, aq)
        t1 = time.perf_counter()
        aq.solve(ref_problem, aq.SolverParams(eps_tol=eps, iter_limit=warmup + steps + 1))
        total = time.perf_counter() - t1
    finally:
        eng.pdhg_step = inner_step
        eng.estimate_norm = orig_norm
    if len(starts) < warmup + steps + 1:
        raise RuntimeError(f"reference finished early ({len(starts)} outer iterations)")
    seconds = starts[warmup + steps] - starts[warmup]
    return dict(kind="reference", backend=aq.active_backend(), seconds=seconds,
                inner=int(sum(inners[warmup:warmup + steps])), outer=steps, total_seconds=total,
                convert_seconds=t1 - t0, init_seconds=starts[0] - t1 if starts else None, spec=spec)


def _run_port(problem, warmup, steps, eps, spec):
    import oracle
    from paper_2602_23967_b200 import SolverParams

    # the oracle has no per-step hook: time whole bounded solves
    t0 = time.perf_counter()
    r0 = oracle.solve(problem, SolverParams(eps_tol=eps, iter_limit=warmup))
    t1 = time.perf_counter()
    r1 = oracle.solve(problem, SolverParams(eps_tol=eps, iter_limit=warmup + steps))
    t2 = time.perf_counter()
    return dict(kind="port", backend="oracle-port", seconds=(t2 - t1) - (t1 - t0),
                inner=int(r1["inner"] - r0["inner"]), outer=steps, total_seconds=t2 - t0, spec=spec)


def run(spec: str, warmup: int, steps: int, eps: float = 1e-8):
    import instances

    return run_problem(instances.build(spec), warmup, steps, eps, spec)


if __name__ == "__main__":
    spec, w, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    print(json.dumps(run(spec, w, k)))
