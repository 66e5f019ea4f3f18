"""Compare per-check traces of ours vs the reference to locate divergence."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import refbridge
aq = refbridge.load_reference()
import paper_2602_23967_b200 as ours

def trace(mod, p, **kw):
    tr = []
    r = mod.solve(p, mod.SolverParams(**kw), progress=lambda it, rep, om, rd: tr.append((it, rep.r_primal, rep.r_dual, rep.r_gap, om, rd)))
    return r, tr

for args, kw in [((40, 20, "diagonal", 0.3, 1), dict(eps_tol=1e-8)), ((40, 20, "diagonal", 0.3, 1), dict(eps_tol=1e-8, check_every=1, iter_limit=400)),
                 ((30, 15, "low_rank", 0.3, 4), dict(eps_tol=1e-8, check_every=1, iter_limit=300))]:
    p = ours.random_qp(*args)
    r1, t1 = trace(ours, p, **kw)
    r0, t0 = trace(aq, refbridge.to_reference(p, aq), **kw)
    print(args, kw, "ours", r1.outer_iterations, "ref", r0.outer_iterations)
    first = None
    for a, b in zip(t1, t0):
        rel = max(abs(a[i] - b[i]) / max(abs(b[i]), 1e-300) for i in (1, 2, 3, 4))
        if a[5] != b[5] or rel > 1e-6:
            first = (a, b, rel); break
    print("  first divergence:", first)
    for a, b in list(zip(t1, t0))[:12]:
        print("   ", a[0], ["%.6e" % v for v in a[1:5]], a[5], "|", ["%.6e" % v for v in b[1:5]], b[5])
