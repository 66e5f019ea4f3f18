"""Compare our per-check trace with a golden reference trace; print first divergence."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import instances
import paper_2602_23967_b200 as ours
for spec in sys.argv[1:]:
    g = json.load(open(os.path.join(ROOT, "tests/golden", "ref_" + spec.replace(":", "_") + ".json")))
    tr = []
    r = ours.solve(instances.build(spec), ours.SolverParams(eps_tol=g["eps_tol"]),
                   progress=lambda it, rep, om, rd: tr.append([it, rep.r_primal, rep.r_dual, rep.r_gap, om, rd]))
    print(spec, "ours", r.status.value, r.outer_iterations, r.inner_iterations, r.restarts, "ref", g["status"], g["outer"], g["inner"], g["restarts"])
    for a, b in zip(tr, g["trace"]):
        rel = max(abs(a[i] - b[i]) / max(abs(b[i]), 1e-300) for i in (1, 2, 3, 4))
        if a[0] != b[0] or a[5] != b[5] or rel > 1e-6:
            print("  diverge at", a, "\n        ref", b, "rel", rel)
            break
    else:
        print("  traces agree over", min(len(tr), len(g["trace"])), "checks")
