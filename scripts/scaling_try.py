"""Opt-in Ruiz / Pock-Chambolle scaling vs the unscaled (reference) solve."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import instances
import paper_2602_23967_b200 as aq
specs = sys.argv[1:] or ["c1:0", "rqp:300:150:sparse:0.05:7", "rqp:500:300:diagonal:0.02:5",
                         "rqp:300:150:low_rank:0.05:3", "c4u:1e3:1", "c4i:1e3:1", "c2:1e4:5e3:0", "c3:2e3:100:0"]
for spec in specs:
    p = instances.build(spec)
    line = f"{spec:30s}"
    for sc in (None, "ruiz", "ruiz_pc"):
        t = time.time()
        r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, scaling=sc, iter_limit=200000))
        line += (f" | {sc or 'none'}: {r.status.value} {r.outer_iterations}/{r.inner_iterations} "
                 f"obj={r.report.primal_objective:.10g} kkt={r.report.kkt_max:.1e} {time.time()-t:.2f}s")
    print(line, flush=True)
