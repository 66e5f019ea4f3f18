"""Device-trace breakdown of the C2 window graph (AQP_TRACE=1)."""
import os, sys, collections
os.environ["AQP_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators, engine, _native as nat
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver
p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
prm = aq.SolverParams(eps_tol=1e-8)
dev = DeviceProblem(p, DeviceContext.get(0))
sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0 + p.quad.inf_norm_bound(), tol_scale=5e-4,
                   tol_floor=1e-9, diag_bound=p.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
eta = engine.estimate_eta(sol, p, prm)
sc = nat.Scalars(); sc.eta, sc.omega, sc.inner_tol = eta, 1.0, 1e-6   # tight tol: many BB iterations
sol.init(sc)
print("pdl", sol.uses_pdl())
sol.trace()
for w in range(3):
    sol.run(64)
    s = sol.get_scalars()
print("last window: outer", s.iters_done, "inner", s.inner_sum)
tr = sol.trace()
names = {}
def name(tag):
    kind, grid = int(tag) >> 32, int(tag) & 0xffffffff
    return f"{['spmv','elem','fin0','fin1','folded','finalized'][kind]}/{grid}"
seq = [(name(t), int(ns)) for t, ns in tr]
# keep the last window only (events after the last restart of counting are mixed; fine)
trans = collections.defaultdict(list)
for (a, ta), (b, tb) in zip(seq, seq[1:]):
    trans[(a, b)].append((tb - ta) / 1e3)
tot = (seq[-1][1] - seq[0][1]) / 1e3
print(f"events {len(seq)} span {tot:.0f} us")
for (a, b), v in sorted(trans.items(), key=lambda kv: -sum(kv[1])):
    v = np.array(v)
    print(f"{a:>14s} -> {b:<14s} n={len(v):6d} mean {v.mean():8.2f} us  median {np.median(v):8.2f}  total {v.sum()/1e3:8.2f} ms")
