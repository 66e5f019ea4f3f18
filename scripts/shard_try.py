"""Quick GPU check of the row-sharded path (virtual ranks on one device)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import shard, generators

def cmp(name, p, prm, ranks):
    t = time.time()
    ref = aq.solve(p, prm)
    t1 = time.time()
    print(f"{name} single: {ref.status.value} outer={ref.outer_iterations} inner={ref.inner_iterations} "
          f"obj={ref.report.primal_objective:.12g} ({t1-t:.1f}s)", flush=True)
    for P in ranks:
        t = time.time()
        rs = shard.solve_local(p, prm, nranks=P, timeout=60)
        r = rs[0]
        same = all(np.array_equal(r.x, q.x) and q.outer_iterations == r.outer_iterations for q in rs)
        print(f"{name} P={P}: {r.status.value} outer={r.outer_iterations} inner={r.inner_iterations} "
              f"obj={r.report.primal_objective:.12g} ranks_identical={same} ({time.time()-t:.1f}s)", flush=True)

prm = aq.SolverParams(eps_tol=1e-8)
cmp("rqp_sparse", aq.random_qp(300, 150, "sparse", density=0.05, seed=7), prm, [1, 2, 3])
cmp("rqp_diag", aq.random_qp(500, 300, "diagonal", density=0.02, seed=5), prm, [2, 4])
cmp("c1", aq.random_qp(2000, 1000, "sparse", density=0.01, seed=0), prm, [2, 8])
