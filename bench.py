"""Benchmark of the PDHCG-II solve loop; headline on BASELINE config 5 (C5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (the largest config BASELINE.json runs on one GPU, and the
one it row-partitions over 1/2/4/8 GPUs): **C5** = ``banded_qp(n=m=5e7,
half_width=5000, seed=0)`` -- A with 5e8 nonzeros (10 per row, banded-local
columns), Q = D + S with 2.5e8 nonzeros in its full symmetric form -- solved
through the public ``paper_2602_23967_b200.solve`` from host (numpy) arrays
with eps_tol = 1e-8 and the reference's default parameters.

* A *step* is one outer PDHG iteration of that solve, with its full BB inner
  solve (A'y pass, BB iterations, x-bar, A x-bar pass, Halpern, window sums).
  Outer iterations [0, W) are warm-up; [W, W+K) are timed with CUDA events on
  the solver stream (the window graphs are split at W and W+K by
  ``solve(..., marks=...)``; splitting does not change the trajectory).  The
  reference arm times the SAME outer iterations [W, W+K) of the same solve of
  the same instance, so both arms measure identical work.
* ``value`` = BB inner iterations / s over the timed outer iterations
  ("CG-inner iters/s" of BASELINE.json; the reference's inner solver is BB,
  SURVEY.md §0), max-over-ranks device time.
* ``e2e`` = the same metric over the WHOLE ``solve`` call (iter_limit = W+K)
  from host buffers: problem upload (H2D), A'/Q build, norm estimate, the W+K
  iterations, the final check and the read-back of x, y (D2H); the timed call
  follows one untimed warm-up call of the same solve (steady state).
* ``roofline``: the dominant kernel of a C5 outer iteration (the BB gradient
  pass: Q SpMV + gradient epilogue + 7 reductions, run 1 + t times per outer
  iteration) timed stand-alone; algorithmic bytes per launch from SURVEY.md
  §8(d) (12 B/nnz + 4 B/row + 64 B/entry).
* ``cpu_baseline``: the reference solver (oracle/_ref, Cython) in this
  process on one core, one outer iteration of the same C5 solve (rank 0,
  N = 1).
* Secondary keys: ``c3_solve`` (config 3, n = 5e6 factor-model portfolio,
  solved to 1e-8) and ``c2_solve`` (config 2, n = 1e6 Lasso-style QP, solved
  to 1e-8), each a full solve timed end to end.

N > 1 (torchrun): ONE C5 solve row-sharded over the N GPUs (SURVEY.md §8(e),
paper_2602_23967_b200/shard.py) -- strong scaling of the same workload and
step range; ``value`` is that solve's BB iterations / s over [W, W+K)
(max-over-ranks device time).  ``--impl reference`` times the reference CPU
solver (rank 0 only) on the same workload, range and metric.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C5_N, C5_W = 50_000_000, 5000
# test hooks only (scripts/bench_dist_try.sh, tests): a smaller instance and
# the gloo backend with ranks sharing one device -- never used by the driver
_TEST_N = int(os.environ.get("AQP_BENCH_TEST_N", "0"))
_SKIP_SECONDARY = os.environ.get("AQP_BENCH_NO_SECONDARY", "") == "1"
EPS = 1e-8
METRIC = "BB(CG)-inner iterations/s, C5 solve to 1e-8 rel. KKT (outer iterations [W, W+K))"
HBM_PEAK_FALLBACK = 6650.0


def c5_dims():
    n = _TEST_N or C5_N
    w = C5_W if not _TEST_N else max(50, min(C5_W, _TEST_N // 100))
    return n, w


def c5_problem():
    from paper_2602_23967_b200 import generators

    n, w = c5_dims()
    return generators.banded_qp(n, n, half_width=w, seed=0)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampler over the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sms = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        busy = [s for s in sms if s > 300] or sms
        busy.sort()
        return {"sm_mhz": busy[len(busy) // 2] if busy else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("AQP_BENCH_TEST_BACKEND", "nccl"))
    return world, rank, local


def q_full_nnz(p) -> int:
    q = p.quad if p.quad.kind == "sparse" else getattr(p.quad, "p", None)
    if q is None:
        return 0
    up = q.upper
    diag_stored = int(np.count_nonzero(np.asarray(up.indices) == np.repeat(np.arange(p.n), np.diff(up.indptr))))
    return 2 * up.nnz - diag_stored


def workload_name(p) -> str:
    n, w = c5_dims()
    return (f"C5 banded sparse QP n=m={p.n} half_width={w} seed=0 nnz(A)={p.constraint_matrix.nnz} "
            f"nnz(Q_full)={q_full_nnz(p)} (BASELINE configs[4]: the largest 1-GPU config, row-partitioned for N>1)")


def problem_bytes(p) -> int:
    a, q = p.constraint_matrix, p.quad
    arrs = [a.indptr, a.indices, a.data, p.cost, p.var_bounds.lower, p.var_bounds.upper, p.con_bounds.lower,
            p.con_bounds.upper]
    if q.kind == "diagonal":
        arrs.append(q.values)
    else:
        pq = q if q.kind == "sparse" else q.p
        arrs += [pq.upper.indptr, pq.upper.indices, pq.upper.data, pq.diag]
        if q.kind == "sparse_low_rank":
            arrs += [q.r.indptr, q.r.indices, q.r.data]
    return int(sum(np.asarray(x).nbytes for x in arrs))


def host_cpu() -> dict:
    """nproc and the CPU model of the box the reference timing ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def ref_sample(problem, warmup: int, steps: int, threads: int):
    """Reference CPU solver on outer iterations [warmup, warmup+steps) of the same solve."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_bench

    if threads == 1:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(limits=1):
            return ref_bench.run_problem(problem, warmup, steps, EPS)
    return ref_bench.run_problem(problem, warmup, steps, EPS)


def base_line(args, world, value, ms, sharded):
    return {
        "metric": METRIC, "value": value, "unit": "inner_iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps if args.steps else None, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
    }


def config_block(problem, args, world, sharded):
    return {"workload": workload_name(problem),
            "range": f"outer iterations [{args.warmup}, {args.warmup + args.steps}) of one solve from the "
                     f"reference's initial point (both arms)",
            "step": "one outer PDHG iteration incl. its full BB inner solve",
            "eps_tol": EPS, "params": "reference defaults (SolverParams(eps_tol=1e-8))",
            "parallelism": f"rowshard{world}" if sharded else ("replicas" if world > 1 else "single"),
            "l2": "inputs (~10 GB of matrices + vectors per BB iteration) are ~80x the 126 MB L2: no flush needed; "
                  "stand-alone kernel timings flush L2 anyway"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    t0 = time.perf_counter()
    problem = c5_problem()
    gen_s = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    r = ref_sample(problem, args.warmup, args.steps, threads)
    value = r["inner"] / r["seconds"]
    line = base_line(args, args.gpus, value, 1e3 * r["seconds"], args.gpus > 1)
    # the same config block as the GPU arm (same workload, range and params):
    # how the reference executes is described in cpu_baseline
    line["config"] = config_block(problem, args, args.gpus, args.gpus > 1)
    line.update({
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "inner_iters/s", "cores": threads, "kind": r["kind"], **host_cpu(),
                         "sample": f"outer iterations [{args.warmup}, {args.warmup + args.steps}) of the C5 solve "
                                   f"({r['inner']} BB iterations in {r['seconds']:.1f}s; backend {r['backend']}: "
                                   f"single-threaded Cython kernels, numpy/OpenBLAS with {threads} threads; "
                                   f"instance generation {gen_s:.0f}s, conversion {r.get('convert_seconds', 0):.0f}s "
                                   f"and initialisation {r.get('init_seconds') or 0:.0f}s untimed)"},
        "e2e": {"value": value, "unit": "inner_iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(line), flush=True)


def kernel_table(problem, local, kinds):
    """Stand-alone event timing of the hot kernels on a fresh solver of `problem`."""
    import torch

    from paper_2602_23967_b200 import _native as nat
    from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver

    n, m = problem.n, problem.m
    dev = DeviceProblem(problem, DeviceContext.get(local))
    sol = DeviceSolver(dev, eps_tol=EPS, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                       diag_bound=problem.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
    sc = nat.Scalars()
    sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
    sol.init(sc)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    info = dev.info
    nnz_q = info.q_full_nnz
    table = {
        "bb_gradient": (0, 12 * nnz_q + 4 * (n + 1) + 64 * n),
        "bb_step": (1, 40 * n),
        "p1_At_y": (2, 12 * info.at_nnz + 4 * (n + 1) + 8 * m + 40 * n),
        "p2_A_xbar": (3, 12 * info.a_nnz + 4 * (m + 1) + 8 * n + 48 * m),
        "x_post": (4, 48 * n),
        "bb_fold": (5, 8 * 7 * max(info.q_items, 1)),
    }
    out = {}
    for name in kinds:
        kid, nbytes = table[name]
        sol.time_kernel(kid, 2, flush)
        avg = sol.time_kernel(kid, 10, flush)
        out[name] = {"ms": avg, "alg_bytes": int(nbytes), "gbs": nbytes / (avg * 1e-3) / 1e9}
    fixed, per_inner = sol.counters()
    del sol, dev, flush
    gc.collect()
    torch.cuda.empty_cache()
    return out, fixed, per_inner


def full_solve_key(problem, local, name):
    """One full solve to 1e-8 from host arrays, timed end to end."""
    import torch

    import paper_2602_23967_b200 as aq

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = aq.solve(problem, aq.SolverParams(eps_tol=EPS), device=local)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"workload": name, "status": res.status.value, "outer": res.outer_iterations,
           "inner": res.inner_iterations, "restarts": res.restarts, "kkt": res.report.kkt_max,
           "objective": res.report.primal_objective, "solve_time_s": wall,
           "inner_iters_per_s": res.inner_iterations / wall, "outer_iters_per_s": res.outer_iterations / wall}
    del res
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_ours(args, world, rank, local):
    import torch

    import paper_2602_23967_b200 as aq

    local = local % torch.cuda.device_count()  # ranks > devices only in the one-box test hook
    torch.cuda.set_device(local)
    sharded = world > 1
    t0 = time.perf_counter()
    problem = c5_problem()
    gen_s = time.perf_counter() - t0
    group = None
    if sharded:
        from paper_2602_23967_b200.shard import DistGroup

        group = DistGroup()
    n, m = problem.n, problem.m
    stream = torch.cuda.current_stream()
    marks = {}
    W, K = args.warmup, args.steps
    clocks = Clocks(local)

    def monitor(outer, inner):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        marks[outer] = (ev, inner)

    # runtime initialisation outside the timed region (a serving process holds
    # it): the libaqp context on this stream, incl. its pinned staging pool
    from paper_2602_23967_b200.device import DeviceContext

    DeviceContext.get(local)
    # one untimed warm-up call of the same solve (the first call of a process
    # also pays the device allocator's first mappings of ~15 GB and the first
    # touch of the staging path: 1.1 s of upload instead of 0.3 s, AQP_PHASES);
    # the timed call below is the steady state of a serving process
    aq.solve(problem, aq.SolverParams(eps_tol=EPS, iter_limit=W + K), device=local, group=group)
    gc.collect()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # clocks are sampled over the whole solve call (it contains the timed
    # region, ~0.26 s on C5: too short for a sampler started inside it)
    clocks.start()
    time.sleep(0.3)  # nvidia-smi is up before the GPU work begins
    t0 = time.perf_counter()
    res = aq.solve(problem, aq.SolverParams(eps_tol=EPS, iter_limit=W + K), device=local, monitor=monitor,
                   group=group, marks=[W, W + K])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    clk["scope"] = "nvidia-smi every 50 ms over the whole solve call, which contains the timed region"
    ms = marks[W][0].elapsed_time(marks[W + K][0])
    inner = marks[W + K][1] - marks[W][1]
    t = torch.tensor([ms, wall], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max, wall_max = t[0].item(), t[1].item()
    value = inner / (ms_max / 1e3)  # one solve: every rank reports the same counts
    e2e_value = res.inner_iterations / wall_max
    result = {"status": res.status.value, "outer": res.outer_iterations, "inner": res.inner_iterations,
              "kkt": res.report.kkt_max, "objective": res.report.primal_objective}
    del res
    gc.collect()
    torch.cuda.empty_cache()
    if group is not None:
        group.close()
    if rank != 0:
        return

    peak, peak_kind = peaks()
    kernels, fixed, per_inner = kernel_table(problem, local, ("bb_gradient", "bb_step", "p1_At_y", "p2_A_xbar",
                                                              "x_post", "bb_fold"))
    top = kernels["bb_gradient"]
    traffic = None  # ncu dram__bytes_{read,write}.sum of the same kernel (scripts/profile_r02.sh)
    for prof in ("ncu_summary_r02e.json", "ncu_summary_r02.json", "ncu_summary.json"):
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", prof)))["kernels"]["c5_bb_gradient"][
                "dram_bytes_per_launch"]
            break
        except Exception:
            traffic = None
    nnz_q = q_full_nnz(problem)
    nnz_a = problem.constraint_matrix.nnz
    # algorithmic bytes of the timed range (SURVEY.md §8(d) pass model)
    b_in = 12 * nnz_q + 4 * (n + 1) + 112 * n
    b_out_fixed = 24 * nnz_a + 4 * (n + m + 2) + 80 * n + 64 * m + b_in - 24 * n
    alg_gbs = (K * b_out_fixed + inner * b_in) / (ms_max / 1e3) / 1e9
    line = base_line(args, world, value, ms_max, sharded)
    line["config"] = config_block(problem, args, world, sharded)
    line.update({
        "timed": {"outer": K, "inner": inner, "ms": ms_max, "inner_per_outer": inner / max(K, 1),
                  "outer_iters_per_s": K / (ms_max / 1e3), "alg_gbs": alg_gbs, "alg_frac": alg_gbs / peak},
        "solve": dict(result, iter_limit=W + K, wall_s=wall_max, gen_s=gen_s),
        "e2e": {"value": e2e_value, "unit": "inner_iters/s", "h2d_bytes_per_step": problem_bytes(problem),
                "d2h_bytes_per_step": 8 * (2 * n + m),
                "scope": f"one e2e step = one whole solve call from host (numpy) arrays with iter_limit {W + K}: "
                         f"staged H2D of the problem, device validation and A'/Q/SELL build, norm estimate, all "
                         f"{W + K} outer iterations, final check, D2H of x, y and the dual slack; value = its BB "
                         f"iterations / its wall time (libaqp context created and one untimed warm-up call of the same solve "
                         f"before the timer)"},
        "roofline": {"bound": "hbm", "achieved": top["gbs"], "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": top["gbs"] / peak, "traffic": traffic,
                     "kernel": "C5 bb_gradient (Q SpMV + gradient epilogue + 7 sums)",
                     "alg_bytes_per_launch": top["alg_bytes"], "ms_per_launch": top["ms"],
                     "alg_bytes_rule": "12*nnz(Q_full) + 4*(n+1) + 64*n (SURVEY.md §8(d))"},
        "kernels": kernels,
        "gpu_launches": int(K * fixed + inner * per_inner),
        "clocks": clk,
    })
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = ref_sample(problem, 1, 1, threads=1)
            line["cpu_baseline"] = {"value": cb["inner"] / cb["seconds"], "unit": "inner_iters/s", "cores": 1,
                                    "kind": cb["kind"], **host_cpu(),
                                    "sample": f"outer iteration [1, 2) of the same C5 solve ({cb['inner']} BB "
                                              f"iterations in {cb['seconds']:.1f}s, backend {cb['backend']}, "
                                              f"1 BLAS thread)"}
        except Exception as exc:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(exc)[-300:]}
    del problem
    gc.collect()
    if world == 1 and not _SKIP_SECONDARY:
        from paper_2602_23967_b200 import generators

        p3 = generators.portfolio_qp(5_000_000, 100, seed=0)
        line["c3_solve"] = full_solve_key(p3, local, "C3 factor-model portfolio n=5e6 k=100 (BASELINE configs[2])")
        del p3
        p2 = generators.lasso_style_qp(1_000_000, 500_000, seed=0)
        line["c2_solve"] = full_solve_key(p2, local, "C2 Lasso-style QP n=1e6 m=5e5 (BASELINE configs[1])")
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 or args.steps < 1:
        ap.error("need --warmup >= 3 and --steps >= 1")
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
