"""Short C2 run for profiling (2 certification windows)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators
p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
it = int(sys.argv[1]) if len(sys.argv) > 1 else 128
r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, iter_limit=it))
print(r.status.value, r.outer_iterations, r.inner_iterations)
