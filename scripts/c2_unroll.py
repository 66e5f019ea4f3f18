"""C2 solve time vs BB-loop unroll (AQP_BB_UNROLL, read at solver creation)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators

p = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
for u in sys.argv[1:]:
    os.environ["AQP_BB_UNROLL"] = u
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = aq.solve(p, aq.SolverParams(eps_tol=1e-8))
    torch.cuda.synchronize()
    print(json.dumps({"unroll": int(u), "s": round(time.perf_counter() - t, 2), "status": r.status.value,
                      "outer": r.outer_iterations, "inner": r.inner_iterations}), flush=True)
