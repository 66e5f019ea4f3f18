"""Stand-alone timings (L2 flushed) of the C3 low-rank passes: dense R x (+ fold)
and R'(R x) on the 100 x 5e6 dense factor, and the gradient pass over P.

    python scripts/c3_kernels.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_23967_b200 import _native as nat, generators  # noqa: E402
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver  # noqa: E402

p = generators.portfolio_qp(5_000_000, 100, seed=0)
dev = DeviceProblem(p, DeviceContext.get(0))
sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                   diag_bound=p.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
sc = nat.Scalars()
sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
sol.init(sc)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
n, k = p.n, 100
alg = {6: 8 * k * n + 8 * n, 7: 8 * k * n + 8 * n, 0: None, 1: 40 * n}
out = {}
for kid, name in ((6, "dense_rx+fold"), (7, "dense_rtv"), (0, "gradient(P)"), (1, "bb_step")):
    sol.time_kernel(kid, 2, flush)
    ms = sol.time_kernel(kid, 10, flush)
    out[name] = {"ms": round(ms, 4)}
    if alg[kid]:
        out[name]["gbs"] = round(alg[kid] / (ms * 1e-3) / 1e9, 1)
print(json.dumps(out))
