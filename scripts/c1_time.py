"""Median solve time of small instances (C1 family, C4 n=1e4) -- latency-bound windows."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch
import instances
import paper_2602_23967_b200 as aq
out = {}
for spec in sys.argv[1:] or ["c1:0", "c1:1", "c4i:1e4:1", "c2:1e4:5e3:0"]:
    p = instances.build(spec)
    prm = aq.SolverParams(eps_tol=1e-8)
    aq.solve(p, prm)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = aq.solve(p, prm)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    out[spec] = {"median_s": round(sorted(ts)[2], 4), "outer": r.outer_iterations, "inner": r.inner_iterations}
print(json.dumps(out))
