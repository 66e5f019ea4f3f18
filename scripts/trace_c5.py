"""Device-trace breakdown of C5 outer iterations (AQP_TRACE=1): where one step's
time goes between and inside the window graph's kernels.

    python scripts/trace_c5.py [n] [outer]
"""
import collections
import os
import sys

os.environ["AQP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2602_23967_b200 as aq  # noqa: E402
from paper_2602_23967_b200 import _native as nat, engine, generators  # noqa: E402
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 50_000_000
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = generators.banded_qp(n, n, half_width=5000 if n >= 5_000_000 else max(50, n // 100), seed=0)
prm = aq.SolverParams(eps_tol=1e-8)
dev = DeviceProblem(p, DeviceContext.get(0))
info = dev.setup_info()
sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0 + info.q_bound, tol_scale=5e-4, tol_floor=1e-9,
                   diag_bound=info.diag_bound, adaptive=True, max_inner=200, halpern=True)
eta = engine.estimate_eta(sol, p, prm)
sc = nat.Scalars()
sc.eta, sc.omega, sc.inner_tol = eta, 1.0, 1e-2
sol.init(sc)
sol.run(5)
sol.get_scalars()
sol.trace()
sol.run(outer)
s = sol.get_scalars()
print("outer", s.iters_done, "inner", s.inner_sum)
tr = sol.trace()


def name(tag):
    kind, grid = int(tag) >> 32, int(tag) & 0xffffffff
    return f"{['spmv', 'elem', 'fin0', 'fin1', 'folded', 'finalized'][kind]}/{grid}"


seq = [(name(t), int(ns)) for t, ns in tr]
trans = collections.defaultdict(list)
for (a, ta), (b, tb) in zip(seq, seq[1:]):
    trans[(a, b)].append((tb - ta) / 1e3)
tot = (seq[-1][1] - seq[0][1]) / 1e3
print(f"events {len(seq)} span {tot:.0f} us = {tot / max(s.iters_done, 1):.0f} us per outer iteration")
for (a, b), v in sorted(trans.items(), key=lambda kv: -sum(kv[1])):
    v = np.array(v)
    print(f"{a:>14s} -> {b:<14s} n={len(v):6d} mean {v.mean():9.2f} us  median {np.median(v):9.2f}  "
          f"total {v.sum() / 1e3:8.2f} ms")
