"""Set up a solver on a named config and launch hot kernels stand-alone (for ncu).
    python scripts/prof_kernel.py c5 3 [reps]      # kernel ids as aqp_solver_time_kernel"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
from bench_configs import build
from paper_2602_23967_b200 import _native as nat
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver

name = sys.argv[1]
kids = [int(k) for k in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = build(name)
dev = DeviceProblem(p, DeviceContext.get(0))
sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                   diag_bound=p.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
sc = nat.Scalars(); sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
sol.init(sc)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
for kid in kids:
    print(kid, sol.time_kernel(kid, reps, flush))
