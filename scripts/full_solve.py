"""Full-scale solve of a named BASELINE config to 1e-8 on one B200 (evidence run).
    python scripts/full_solve.py c3|c5|c5d [time_limit_s]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
import paper_2602_23967_b200 as aq
from bench_configs import build

name = sys.argv[1]
tl = float(sys.argv[2]) if len(sys.argv) > 2 else 1200.0
scaling = sys.argv[3] if len(sys.argv) > 3 else None
t = time.time()
p = build(name)
gen = time.time() - t
trace = []
t = time.time()


def progress(k, rep, om, rd):
    trace.append((k, rep.kkt_max, om))
    if len(trace) % 20 == 1:  # partial evidence survives a killed run
        print(json.dumps({"outer": k, "kkt": rep.kkt_max, "omega": om, "round": rd, "s": round(time.time() - t, 1)}),
              file=sys.stderr, flush=True)


res = aq.solve(p, aq.SolverParams(eps_tol=1e-8, time_limit=tl, scaling=scaling), progress=progress)
torch.cuda.synchronize()
wall = time.time() - t
print(json.dumps({"config": name, "scaling": scaling, "n": p.n, "m": p.m, "status": res.status.value, "outer": res.outer_iterations,
                  "inner": res.inner_iterations, "restarts": res.restarts, "kkt": res.report.kkt_max,
                  "objective": res.report.primal_objective, "solve_s": round(wall, 2), "gen_s": round(gen, 1),
                  "outer_per_s": round(res.outer_iterations / wall, 1),
                  "inner_per_s": round(res.inner_iterations / wall, 1),
                  "kkt_trace": [(k, float(f"{v:.3e}")) for k, v, _ in trace[:: max(1, len(trace) // 40)]]}))
