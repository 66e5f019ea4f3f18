"""Per-config throughput + roofline on one B200 for BASELINE.json configs 2, 3, 5
(C2 lasso n=1e6, C3 portfolio n=5e6 k=100 dense factor, C5 banded n=m=5e7).

For each config: a bounded solve (W warm-up + K timed certification windows of
64 outer iterations, CUDA events on the solver stream via the monitor hook)
and stand-alone kernel timings (L2 flushed before each launch) with the
algorithmic bytes of SURVEY.md §8(d).  Prints one JSON object per config.

    python scripts/bench_configs.py c3 c5 [--windows K] [--warmup W]
"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver
from paper_2602_23967_b200 import _native as nat


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def build(name):
    if name == "c2":
        return generators.lasso_style_qp(1_000_000, 500_000, seed=0)
    if name == "c3":
        return generators.portfolio_qp(5_000_000, 100, seed=0)
    if name == "c5":
        return generators.banded_qp(50_000_000, 50_000_000, half_width=5000, seed=0)
    if name == "c5d":
        return generators.banded_qp(50_000_000, 50_000_000, half_width=5000, seed=0, diagonal_q=True)
    raise ValueError(name)


def run(name, W, K):
    t0 = time.time()
    p = build(name)
    gen_s = time.time() - t0
    n, m = p.n, p.m
    nnz_a = p.constraint_matrix.nnz
    stream = torch.cuda.current_stream()
    marks = {}

    def monitor(outer, inner):
        idx = outer // 64
        if idx in (W, W + K):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            marks[idx] = (ev, outer, inner)

    prm = aq.SolverParams(eps_tol=1e-8, iter_limit=64 * (W + K))
    t1 = time.time()
    res = aq.solve(p, prm, monitor=monitor)
    torch.cuda.synchronize()
    solve_s = time.time() - t1
    ms = marks[W][0].elapsed_time(marks[W + K][0])
    outer = marks[W + K][1] - marks[W][1]
    inner = marks[W + K][2] - marks[W][2]
    # per-kernel stand-alone timings
    dev = DeviceProblem(p, DeviceContext.get(0))
    info = dev.info
    q = p.quad
    sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                       diag_bound=q.diag_bound(), adaptive=True, max_inner=200, halpern=True)
    sc = nat.Scalars(); sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
    sol.init(sc)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    nq = info.q_full_nnz
    k = q.r.rows if q.kind == "sparse_low_rank" else 0
    ks = {"p1_At_y": (2, 12 * info.at_nnz + 4 * (n + 1) + 8 * m + (88 if q.kind == "diagonal" else 24) * n),
          "p2_A_xbar": (3, 12 * nnz_a + 4 * (m + 1) + 8 * n + 48 * m)}
    if q.kind != "diagonal":
        ks["bb_gradient"] = (0, 12 * nq + 4 * (n + 1) + 64 * n + (8 * n if k else 0))
        ks["bb_step"] = (1, 40 * n)
        ks["x_post"] = (4, 48 * n)
    if k and info.r_dense:
        ks["dense_Rx"] = (6, 8 * k * n + 8 * n)
        ks["dense_Rtv"] = (7, 8 * k * n + 8 * n)
    kern = {}
    for nm, (kid, nbytes) in ks.items():
        sol.time_kernel(kid, 2, flush)
        t = sol.time_kernel(kid, 10, flush)
        kern[nm] = {"us": round(t * 1e3, 2), "alg_MB": round(nbytes / 1e6, 1), "gbs": round(nbytes / t / 1e6, 1),
                    "frac": round(nbytes / t / 1e6 / peak(), 3)}
    print(json.dumps({"config": name, "n": n, "m": m, "nnz_A": nnz_a, "nnz_Q_full": nq, "k": k,
                      "r_dense": int(info.r_dense), "gen_s": round(gen_s, 1), "solve_s": round(solve_s, 1),
                      "status": res.status.value, "outer": res.outer_iterations, "inner": res.inner_iterations,
                      "kkt": res.report.kkt_max, "timed_windows": K, "timed_ms": round(ms, 2),
                      "outer_per_s": round(outer / (ms / 1e3), 1), "inner_per_s": round(inner / (ms / 1e3), 1),
                      "inner_per_outer": round(inner / max(outer, 1), 2), "peak_gbs": peak(), "kernels": kern}),
          flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--windows", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    for c in a.configs:
        run(c, a.warmup, a.windows)
