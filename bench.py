"""Benchmark of the PDHCG-II solve loop on BASELINE config 2 (C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N = 1): ``lasso_style_qp(n=1e6, m=5e5, seed)`` -- the Lasso-style
sparse QP with Q = D + S (5e6 nnz full) and A (4e6 nnz) of BASELINE.json
configs[1] -- solved to 1e-8 relative KKT through the public
``paper_2602_23967_b200.solve`` from host (numpy) arrays.

* A *step* is one certification window of that solve: 64 outer PDHG
  iterations, each with its full BB inner solve, plus the certification point
  (device residuals, ray tests, host branch logic).  W windows are warm-up,
  the next K are timed with CUDA events on the solver stream (synchronised on
  both sides by the certification point itself).
* ``value`` = BB inner iterations / s over the K timed windows, summed over
  ranks and divided by the max rank time ("CG-inner iters/s" of BASELINE.json;
  the reference's inner solver is BB).
* ``e2e`` = the same metric over the WHOLE solve call to 1e-8 from host
  buffers: problem upload (H2D), A'/Q build, norm estimate, all iterations,
  and the read-back of x, y (D2H) -- ``solve_time_s`` is that call's wall time.
* ``roofline``: the dominant kernel (BB gradient pass: Q SpMV + gradient
  epilogue + 7 reductions) timed stand-alone with an L2 flush before each
  launch; algorithmic bytes per launch from SURVEY.md §8(d).
* ``cpu_baseline``: the reference solver (oracle/_ref, Cython) on the host,
  1 core, bounded sample of the same solve (rank 0, N = 1).

N > 1 (torchrun): ONE C2 solve row-sharded over the N GPUs (SURVEY.md §8(e),
paper_2602_23967_b200/shard.py): rank r owns a block of rows of A, A' and Q,
the gathered vectors are replicated by NVLink peer stores and every
reduction is a one-block mailbox exchange -- strong scaling of the same
workload; ``value`` is that solve's BB iterations / s (max-over-ranks device
time).  ``--replicas`` instead runs N independent C2 solves (weak scaling).
``--impl reference`` times the reference CPU solver (rank 0 only) on the
same workload and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC_N, SPEC_M = 1_000_000, 500_000
# test hooks only (scripts/bench_dist_try.sh): a smaller instance, an iteration
# cap, the gloo backend and ranks sharing one device -- never used by the driver
_TEST_N = int(os.environ.get("AQP_BENCH_TEST_N", "0"))
_TEST_ITERS = int(os.environ.get("AQP_BENCH_TEST_ITERS", "0"))
CHECK_EVERY = 64
EPS = 1e-8
METRIC = "BB(CG)-inner iterations/s, C2 solve to 1e-8 rel. KKT"
HBM_PEAK_FALLBACK = 6650.0


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
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def workload_name(p) -> str:
    nnz_q = 2 * p.quad.upper.nnz - int(np.count_nonzero(p.quad.upper.indices == np.repeat(
        np.arange(p.n), np.diff(p.quad.upper.indptr))))
    return (f"C2 lasso-style QP n={p.n} m={p.m} nnz(A)={p.constraint_matrix.nnz} nnz(Q_full)={nnz_q} "
            f"(BASELINE configs[1])")


def problem_bytes(p) -> int:
    a, q = p.constraint_matrix, p.quad
    arrs = [a.indptr, a.indices, a.data, p.cost, p.var_bounds.lower, p.var_bounds.upper, p.con_bounds.lower,
            p.con_bounds.upper]
    if q.kind == "diagonal":
        arrs.append(q.values)
    else:
        pq = q if q.kind == "sparse" else q.p
        arrs += [pq.upper.indptr, pq.upper.indices, pq.upper.data, pq.diag]
    return int(sum(x.nbytes for x in arrs))


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


def cpu_baseline(spec: str, warmup: int, steps: int, threads: int):
    env = dict(os.environ)
    if threads == 1:
        env.update(OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "ref_bench.py"), spec, str(warmup), str(steps)],
                         capture_output=True, text=True, env=env, timeout=1800)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(args, world, rank):
    if rank != 0:
        return
    spec = f"c2:{SPEC_N}:{SPEC_M}:0"
    threads = os.cpu_count() or 1
    r = cpu_baseline(spec, max(args.warmup, 1), args.steps, threads)
    value = r["inner"] / r["seconds"]
    from paper_2602_23967_b200 import generators

    prob = generators.lasso_style_qp(SPEC_N, SPEC_M, seed=0)
    workload = workload_name(prob)
    line = {
        "metric": METRIC, "value": value, "unit": "inner_iters/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 and not args.replicas else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload,
                   "step": "one outer PDHG iteration (BB inner solve included) of the reference CPU solver",
                   "eps_tol": EPS},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "inner_iters/s", "cores": threads, "kind": r["kind"], **host_cpu(),
                         "sample": f"outer iterations {max(args.warmup,1)}..{max(args.warmup,1)+args.steps} of the C2 solve "
                                   f"({r['inner']} BB iterations in {r['seconds']:.1f}s; backend {r['backend']})"},
        "e2e": {"value": value, "unit": "inner_iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_2602_23967_b200 as aq
    from paper_2602_23967_b200 import generators
    from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver
    from paper_2602_23967_b200 import _native as nat

    local = local % torch.cuda.device_count()  # ranks > devices only in the one-box test hook
    torch.cuda.set_device(local)
    sharded = world > 1 and not args.replicas
    seed = 0 if sharded else rank
    problem = generators.lasso_style_qp(_TEST_N or SPEC_N, (_TEST_N // 2) or SPEC_M, seed=seed)
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
        idx = outer // CHECK_EVERY
        if idx in (W, W + K):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            marks[idx] = (ev, outer, inner)
            if idx == W:
                clocks.start()

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prm = aq.SolverParams(eps_tol=EPS, iter_limit=_TEST_ITERS) if _TEST_ITERS else aq.SolverParams(eps_tol=EPS)
    res = aq.solve(problem, prm, device=local, monitor=monitor, group=group)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    clk = clocks.stop()
    if W in marks and W + K in marks:
        ms = marks[W][0].elapsed_time(marks[W + K][0])
        inner = marks[W + K][2] - marks[W][2]
        outer = marks[W + K][1] - marks[W][1]
    else:  # solve ended before W+K windows: time the whole run
        ms, inner, outer = wall * 1e3, res.inner_iterations, res.outer_iterations
    t = torch.tensor([ms, inner, res.inner_iterations, wall], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        mx = t.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = t.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        ms_max, inner_sum, inner_total_sum, wall_max = mx[0].item(), sm[1].item(), sm[2].item(), mx[3].item()
        if sharded:  # one solve: every rank reports the same counts
            inner_sum, inner_total_sum = inner, res.inner_iterations
    else:
        ms_max, inner_sum, inner_total_sum, wall_max = ms, inner, res.inner_iterations, wall
    value = inner_sum / (ms_max / 1e3)
    e2e_value = inner_total_sum / wall_max

    # --- the same solve with the opt-in device-side Ruiz + Pock-Chambolle
    # scaling (extension, not the reference's algorithm: reported beside the
    # headline, never as it)
    scaled = None
    if not sharded:
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rs_ = aq.solve(problem, aq.SolverParams(eps_tol=EPS, scaling="ruiz_pc"), device=local)
        torch.cuda.synchronize()
        scaled = {"status": rs_.status.value, "outer": rs_.outer_iterations, "inner": rs_.inner_iterations,
                  "kkt": rs_.report.kkt_max, "objective": rs_.report.primal_objective,
                  "solve_time_s": time.perf_counter() - t1,
                  "note": "SolverParams(scaling='ruiz_pc'): opt-in equilibration, certified on the original problem"}

    # --- dominant-kernel roofline (stand-alone, L2 flushed before each launch)
    peak, peak_kind = peaks()
    dev = DeviceProblem(problem, DeviceContext.get(local))
    sol = DeviceSolver(dev, eps_tol=EPS, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                       diag_bound=problem.quad.diag_bound(), adaptive=True, max_inner=200, halpern=True)
    sc = nat.Scalars()
    sc.eta, sc.omega, sc.inner_tol = 0.5, 1.0, 1e-2
    sol.init(sc)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    nnz_q = dev.info.q_full_nnz
    kernels = {}
    for kid, name, nbytes in ((0, "bb_gradient", 12 * nnz_q + 4 * (n + 1) + 64 * n),
                              (1, "bb_step", 40 * n),
                              (2, "p1_At_y", 12 * dev.info.at_nnz + 4 * (n + 1) + 8 * m + 8 * n + 16 * n + 16 * n),
                              (3, "p2_A_xbar", 12 * dev.info.a_nnz + 4 * (m + 1) + 8 * n + 48 * m),
                              (5, "bb_fold", 8 * 7 * dev.info.q_items)):
        sol.time_kernel(kid, 3, flush)
        avg = sol.time_kernel(kid, 20, flush)
        kernels[name] = {"ms": avg, "alg_bytes": nbytes, "gbs": nbytes / (avg * 1e-3) / 1e9}
    top = kernels["bb_gradient"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof))["kernels"]["bb_gradient"]["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    fixed, per_inner = sol.counters()
    n_checks = res.outer_iterations // CHECK_EVERY + 2
    launches = res.outer_iterations * fixed + res.inner_iterations * per_inner + n_checks * 10
    # algorithmic bytes per outer / inner iteration
    b_in = 12 * nnz_q + 4 * (n + 1) + 112 * n
    b_out_fixed = 24 * problem.constraint_matrix.nnz + 4 * (n + m + 2) + 80 * n + 64 * m + b_in - 24 * n
    alg_gbs = (outer * b_out_fixed + inner * b_in) / (ms / 1e3) / 1e9

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "inner_iters/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K if K else None, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(problem),
                   "step": f"one certification window = {CHECK_EVERY} outer iterations + device check",
                   "eps_tol": EPS,
                   "parallelism": f"rowshard{world}" if sharded else ("replicas" if world > 1 else "single"),
                   "l2": "inputs (~230 MB of matrices+vectors per iteration) exceed the 126 MB L2; "
                         "roofline kernel timed with a 512 MB L2 flush before every launch"},
        "solve": {"status": res.status.value, "outer": res.outer_iterations, "inner": res.inner_iterations,
                  "restarts": res.restarts, "kkt": res.report.kkt_max, "objective": res.report.primal_objective,
                  "solve_time_s": wall},
        "solve_time_s": wall,
        "solve_ruiz_pc": scaled,
        "outer_iters_per_s": outer / (ms / 1e3),
        "window_alg_gbs": alg_gbs,
        "e2e": {"value": e2e_value, "unit": "inner_iters/s", "h2d_bytes_per_step": problem_bytes(problem),
                "d2h_bytes_per_step": 8 * (2 * n + m), "scope": "one full solve call from host arrays per step"},
        "roofline": {"bound": "hbm", "achieved": top["gbs"], "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": top["gbs"] / peak, "traffic": traffic, "kernel": "bb_gradient (Q SpMV + epilogue)",
                     "alg_bytes_per_launch": top["alg_bytes"], "ms_per_launch": top["ms"]},
        "kernels": kernels,
        "gpu_launches": int(launches * K * CHECK_EVERY / max(res.outer_iterations, 1)),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(f"c2:{SPEC_N}:{SPEC_M}:0", 2, 8, threads=1)
            line["cpu_baseline"] = {"value": cb["inner"] / cb["seconds"], "unit": "inner_iters/s", "cores": 1,
                                    "kind": cb["kind"], **host_cpu(),
                                    "sample": f"outer iterations 2..10 of the same C2 solve ({cb['inner']} BB "
                                              f"iterations in {cb['seconds']:.1f}s, backend {cb['backend']})"}
        except Exception as exc:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(exc)[-300:]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent solves instead of one sharded solve")
    args = ap.parse_args()
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
