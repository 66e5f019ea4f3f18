"""A/B timing of a bounded C2 solve (first N outer iterations) under the current env."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators
p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
it = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
aq.solve(p, aq.SolverParams(eps_tol=1e-8, iter_limit=64))  # warm
torch.cuda.synchronize()
t = time.time()
r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, iter_limit=it))
torch.cuda.synchronize()
dt = time.time() - t
print(f"{os.environ.get('TAG','')} outer={r.outer_iterations} inner={r.inner_iterations} {dt:.3f}s "
      f"{1e6*dt/max(r.inner_iterations,1):.1f} us/inner kkt={r.report.kkt_max:.3e}")
