"""Persistent window kernel vs graph windows: bitwise equality and time."""
import os, sys, time, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np, torch
    import instances
    import paper_2602_23967_b200 as aq
    out = {}
    for spec in sys.argv[2:]:
        p = instances.build(spec)
        prm = aq.SolverParams(eps_tol=1e-8)
        aq.solve(p, prm)  # warm (module load, allocator)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = aq.solve(p, prm)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
        dt = sorted(ts)[2]
        out[spec] = dict(status=r.status.value, outer=r.outer_iterations, inner=r.inner_iterations, s=round(dt, 4),
                         xsum=float(np.sum(r.x)), xhash=__import__("hashlib").sha1(r.x.tobytes() + r.y.tobytes()).hexdigest()[:12],
                         obj=r.report.primal_objective)
    print(json.dumps(out))
    sys.exit(0)
specs = ["c1:0", "c1:1", "rqp:300:150:sparse:0.05:7", "rqp:500:300:diagonal:0.02:5", "c4u:1e4:1", "c4i:1e4:1",
         "c2:1e4:5e3:0", "c4u:1e5:1"]
res = {}
modes = [("0", None), ("1", None), ("1", "64"), ("1", "24")]
for mode, grid in modes:
    env = dict(os.environ, AQP_PERSISTENT=mode)
    if grid:
        env["AQP_PERSIST_GRID"] = grid
    o = subprocess.run([sys.executable, __file__, "child"] + specs, capture_output=True, text=True, env=env, timeout=900)
    if o.returncode:
        print(o.stderr[-3000:]); sys.exit(1)
    res[(mode, grid)] = json.loads(o.stdout.strip().splitlines()[-1])
for spec in specs:
    a = res[("0", None)][spec]
    line = f"{spec:30s} graph {a['s']:7.4f}s"
    for key in modes[1:]:
        b = res[key][spec]
        same = (a["xhash"], a["outer"], a["inner"]) == (b["xhash"], b["outer"], b["inner"])
        line += f" | grid {key[1] or 'max'}: {b['s']:7.4f}s x{a['s']/b['s']:4.2f} eq={same}"
    print(line + f"  ({a['status']} {a['outer']}/{a['inner']})")
