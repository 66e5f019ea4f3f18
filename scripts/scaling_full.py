"""Full-size C2 (and C5 twin) with the opt-in scalings: solve time to 1e-8."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch
import instances
import paper_2602_23967_b200 as aq
for spec in sys.argv[1:] or ["c2:1e6:5e5:0", "c5:5e4:500:0"]:
    p = instances.build(spec)
    for sc in (None, "ruiz", "ruiz_pc"):
        torch.cuda.synchronize(); t = time.time()
        r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, scaling=sc, time_limit=400))
        torch.cuda.synchronize()
        print(json.dumps({"spec": spec, "scaling": sc, "status": r.status.value, "outer": r.outer_iterations,
                          "inner": r.inner_iterations, "kkt": r.report.kkt_max,
                          "objective": r.report.primal_objective, "seconds": round(time.time() - t, 2)}), flush=True)
