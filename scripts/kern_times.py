"""Stand-alone kernel timings on C2 (L2 flushed before each launch)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2602_23967_b200 import generators, _native as nat
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver
spec = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
n, m = p.n, p.m
dev = DeviceProblem(p, DeviceContext.get(0))
sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                   diag_bound=p.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
sc = nat.Scalars(); sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
sol.init(sc)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
nq = dev.info.q_full_nnz
out = {}
for kid, name, nbytes in ((0, "bb_gradient", 12 * nq + 4 * (n + 1) + 64 * n), (1, "bb_step", 40 * n),
                          (2, "p1", 12 * dev.info.at_nnz + 4 * (n + 1) + 8 * m + 24 * n),
                          (3, "p2", 12 * dev.info.a_nnz + 4 * (m + 1) + 8 * n + 48 * m), (4, "xpost", 48 * n),
                          (5, "bb_fold", 8 * 7 * dev.info.q_items)):
    sol.time_kernel(kid, 3, flush)
    ms = sol.time_kernel(kid, 30, flush)
    ms_warm = sol.time_kernel(kid, 30, None)
    out[name] = dict(us=round(ms * 1e3, 2), us_l2warm=round(ms_warm * 1e3, 2), gbs=round(nbytes / ms / 1e6, 1))
print(json.dumps(out))
