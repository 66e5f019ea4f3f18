import os, sys, time, json
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/oracle')
import instances, paper_2602_23967_b200 as aq
for spec in sys.argv[1:]:
    p = instances.build(spec)
    t=time.time(); tl = float(os.environ.get("TWIN_TIME_LIMIT", "1500")); r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, time_limit=tl)); 
    print(json.dumps(dict(spec=spec, status=r.status.value, outer=r.outer_iterations, inner=r.inner_iterations, restarts=r.restarts, kkt=r.report.kkt_max, obj=r.report.primal_objective, s=time.time()-t)), flush=True)
