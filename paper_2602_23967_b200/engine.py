"""The solve entry point: host control of the device-resident PDHCG-II loop.

Drop-in for ``anchorqp.solve`` (reference ``anchorqp/engine.py:339-498``):
same parameters, statuses, result object, progress-callback cadence and
branch logic.  The iterations themselves never touch the host: each
certification window (<= ``check_every`` outer iterations, each with its
full BB inner solve) is ONE CUDA-graph launch of libaqp, and the host only
synchronises at certification points to run the reference's decision chain
(optimality, ray tests, stall probe, divergence rollback, restart + PID) on
the device-computed scalars.
"""

from __future__ import annotations

import dataclasses
import enum
import math
import os
import sys
import threading
import time
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as nat
from . import certify
from .certify import Certificate, CertificateKind, ResidualReport
from .device import DeviceContext, DeviceProblem, DeviceSolver
from .model import QpProblem, raise_first_violation, validate_dims

# engine.py:26-49
OMEGA_MIN = 1e-6
OMEGA_MAX = 1e6
PID_INTEGRAL_CLAMP = 10.0
ETA_UNCONSTRAINED = 1e8
DIVERGENCE_FACTOR = 100.0
THETA_BACKOFF_FLOOR = 1e-2
STALL_CHECKS = 8
STALL_IMPROVEMENT = 0.99
PROBE_INNER_TOL = 1e-12  # applied on the device (OpGrad<true>::finalize)


class _Phases:
    """AQP_PHASES=1: device-synchronised wall time per setup / loop phase of a
    solve, printed to stderr (diagnostics of the end-to-end path only)."""

    def __init__(self):
        self.on = os.environ.get("AQP_PHASES", "") == "1"
        self.t = time.perf_counter()
        self.acc = {}

    def __call__(self, name):
        if not self.on:
            return
        import torch

        torch.cuda.synchronize()
        now = time.perf_counter()
        self.acc[name] = self.acc.get(name, 0.0) + now - self.t
        self.t = now

    def dump(self):
        if self.on:
            print("AQP_PHASES " + " ".join(f"{k}={v:.4f}" for k, v in self.acc.items()), file=sys.stderr, flush=True)


class SolveStatus(str, enum.Enum):
    OPTIMAL = "optimal"
    PRIMAL_INFEASIBLE = "primal_infeasible"
    DUAL_INFEASIBLE = "dual_infeasible"
    ITERATION_LIMIT = "iteration_limit"
    TIME_LIMIT = "time_limit"


@dataclasses.dataclass(frozen=True)
class RestartParams:
    """engine.py:60-74."""

    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    max_round_len: int = 2000
    enabled: bool = True

    def __post_init__(self):
        if self.enabled and not 0.0 < self.beta_sufficient < self.beta_necessary < 1.0:
            raise ValueError("restart betas must satisfy 0 < sufficient < necessary < 1")
        if self.max_round_len < 1:
            raise ValueError("max_round_len must be positive")


@dataclasses.dataclass(frozen=True)
class InnerParams:
    """engine.py:77-86."""

    adaptive: bool = True
    initial: float = 1e-2
    scale: float = 5e-4
    floor: float = 1e-9
    fixed_tol: float = 1e-9
    max_inner: int = 200


@dataclasses.dataclass(frozen=True)
class SolverParams:
    """engine.py:89-122 (defaults are the reference code's, not SPEC.md's)."""

    eps_tol: float = 1e-6
    eps_inf: float = 1e-9
    theta: float = 0.0
    eta_scale: float = 0.998
    pid_gains: tuple = (0.5, 0.02, 0.1)
    omega0: float = 1.0
    restart: RestartParams = dataclasses.field(default_factory=RestartParams)
    inner: InnerParams = dataclasses.field(default_factory=InnerParams)
    iter_limit: int = 1_000_000
    time_limit: Optional[float] = None
    check_every: int = 64
    halpern: bool = True
    gamma_sys: Optional[float] = None
    norm_iters: int = 100
    norm_seed: int = 0
    # extension (not in the reference, off by default -- SURVEY.md §0): device-
    # side equilibration before the solve, "ruiz" or "ruiz_pc" (Ruiz rounds,
    # then one Pock-Chambolle l1 pass); termination and certificates stay on
    # the original problem
    scaling: Optional[str] = None
    scaling_iters: int = 10

    def __post_init__(self):
        if self.eps_tol <= 0 or self.eps_inf <= 0:
            raise ValueError("tolerances must be positive")
        if not 0.0 <= self.theta < 1.0:
            raise ValueError("theta must lie in [0, 1)")
        if self.omega0 <= 0:
            raise ValueError("omega0 must be positive")
        if self.iter_limit < 1 or self.check_every < 1:
            raise ValueError("iter_limit and check_every must be positive")
        if self.time_limit is not None and self.time_limit <= 0:
            raise ValueError("time_limit must be positive")
        if self.scaling not in (None, "ruiz", "ruiz_pc") or self.scaling_iters < 0:
            raise ValueError("scaling must be None, 'ruiz' or 'ruiz_pc' with scaling_iters >= 0")


@dataclasses.dataclass(frozen=True)
class SolveResult:
    """engine.py:157-171."""

    status: SolveStatus
    x: np.ndarray
    y: np.ndarray
    report: ResidualReport
    certificate: Optional[Certificate]
    outer_iterations: int
    inner_iterations: int
    restarts: int
    seconds: float

    @property
    def rounds(self) -> int:
        return self.restarts + 1


ProgressCallback = Callable[[int, ResidualReport, float, int], None]


@dataclasses.dataclass
class _Round:
    """Host-side scalars of SolverState (engine.py:125-146) that only change at
    certification points; the per-iteration ones (k, inner tolerance) live in
    the device control block."""

    omega: float
    eta: float
    theta: float
    round: int = 0
    pid_integral: float = 0.0
    pid_last_error: float = 0.0
    best_residual_round_start: float = math.inf
    last_check_kkt: float = math.inf


def restart_decision(k: int, rs: _Round, kkt: float, params: SolverParams) -> bool:
    """engine.py:248-257."""
    if k >= params.restart.max_round_len:
        return True
    base = rs.best_residual_round_start
    if kkt <= params.restart.beta_sufficient * base:
        return True
    if kkt <= params.restart.beta_necessary * base and kkt > rs.last_check_kkt:
        return True
    return False


def pid_update(rs: _Round, dx: float, dy: float, params: SolverParams) -> float:
    """engine.py:260-281 with |x - x_rs|, |y - y_rs| from the device."""
    if dx <= 0.0 or dy <= 0.0 or not (math.isfinite(dx) and math.isfinite(dy)):
        return rs.omega
    error = math.log(rs.omega * dx / dy)
    if not math.isfinite(error):
        return rs.omega
    kp, ki, kd = params.pid_gains
    integral = min(max(rs.pid_integral + error, -PID_INTEGRAL_CLAMP), PID_INTEGRAL_CLAMP)
    log_omega = math.log(rs.omega) - (kp * error + ki * integral + kd * (error - rs.pid_last_error))
    rs.pid_integral = integral
    rs.pid_last_error = error
    return min(max(math.exp(log_omega), OMEGA_MIN), OMEGA_MAX)


class _StartVector:
    """The power iteration's first start vector, drawn exactly as the
    reference draws it (``default_rng(norm_seed).standard_normal(cols)``,
    linalg.py:293-294) on a host thread while the problem uploads -- numpy
    releases the GIL while it fills the array (0.5 s at C5).  Redraws continue
    from the same generator."""

    def __init__(self, cols: int, seed: int):
        self.cols = cols
        self.rng = np.random.default_rng(seed)
        self.v = None
        self.thread = threading.Thread(target=self._draw, daemon=True)
        self.thread.start()

    def _draw(self):
        self.v = self.rng.standard_normal(self.cols)

    def first(self) -> np.ndarray:
        self.thread.join()
        return self.v


def estimate_eta(solver: DeviceSolver, problem: QpProblem, params: SolverParams,
                 start: Optional[_StartVector] = None) -> float:
    """initialize()'s step scale (engine.py:178-183, linalg.py:287-312)."""
    a = problem.constraint_matrix
    if a.nnz == 0:
        return ETA_UNCONSTRAINED
    start = start or _StartVector(a.cols, params.norm_seed)
    for attempt in range(8):
        v = start.first() if attempt == 0 else start.rng.standard_normal(a.cols)
        est, annihilated = solver.estimate_norm(v, params.norm_iters)
        if not annihilated:
            return params.eta_scale / est
    return ETA_UNCONSTRAINED


def _setup_info(dev: DeviceProblem, problem: QpProblem, group):
    """Device validation flags + setup scalars; a row shard combines every
    rank's (flags: or, first inverted index: min, maxima: max) and computes
    R's row sums, which span every rank's columns, on the host."""
    info = dev.setup_info()
    if group is None:
        return info
    ints = ("var_nan", "var_wrong_inf", "con_nan", "con_wrong_inf", "cost_nonfinite", "a_nonfinite", "q_nonfinite")
    maxes = ("con_scale", "cost_inf", "q_bound", "r_one", "diag_bound")
    mine = np.array([getattr(info, f) for f in ints + maxes] + [info.var_first_inverted, info.con_first_inverted],
                    dtype=np.float64)
    rows = np.stack(group.gather(mine))
    for i, f in enumerate(ints):
        setattr(info, f, int(rows[:, i].max()))
    for i, f in enumerate(maxes):
        setattr(info, f, float(rows[:, len(ints) + i].max()))
    for i, f in enumerate(("var_first_inverted", "con_first_inverted")):
        col = rows[:, len(ints) + len(maxes) + i]
        col = col[col >= 0]
        setattr(info, f, int(col.min()) if col.size else -1)
    if problem.quad.kind == "sparse_low_rank" and not info.r_inf_done:
        info.r_inf = float(problem.quad.r.row_abs_sums().max(initial=0.0))  # linalg.py:262
        info.r_inf_done = 1
    return info


class _Run:
    """One solve: device objects + the reference's loop locals."""

    def __init__(self, problem: QpProblem, params: SolverParams, progress, device: int, group=None, ph=None):
        ph = ph or _Phases()
        self.problem = problem
        self.params = params
        self.progress = progress
        ctx = DeviceContext.get(device)
        self.group = group
        self.scaling = getattr(params, "scaling", None)
        if self.scaling is not None and group is not None:
            raise ValueError("scaling is not available for row-sharded solves")
        if group is not None:  # row shard of a multi-GPU solve: this rank's rows only (shard.py)
            from .shard import local_part, plan

            self.dev = DeviceProblem(problem, ctx, part=local_part(problem, plan(problem, group.nranks), group.rank))
        else:
            self.dev = DeviceProblem(problem, ctx)
        if ph.on:
            ph.acc["problem_create"] = self.dev.timing.get("create", 0.0)
            ph.t += self.dev.timing.get("create", 0.0)
            ph("problem_upload")
        # validate()'s data checks and the setup scalars, on the device
        info = _setup_info(self.dev, problem, group)
        raise_first_violation(problem, info)
        q_bound = info.q_bound  # QuadOperator.inf_norm_bound (linalg.py:218-220, 260-263)
        if problem.quad.kind == "sparse_low_rank":
            q_bound = q_bound + info.r_one * info.r_inf
        gamma = params.gamma_sys if params.gamma_sys is not None else 1.0 + q_bound  # certify.py:167-169
        self.gamma_sys = gamma
        self.con_scale = info.con_scale  # certify.py:54-60
        self.cost_inf = info.cost_inf
        ph("setup_scalars")
        ip = params.inner
        diag_bound = info.diag_bound
        self.checker_dev = None
        if self.scaling is not None:
            # iterate on an equilibrated copy; certify on the original (checker)
            self.checker_dev = self.dev
            self.dev = DeviceProblem(problem, ctx)
            self.D, self.E = self.dev.scale(getattr(params, "scaling_iters", 10), self.scaling == "ruiz_pc")
            diag_bound = _scaled_diag_bound(problem.quad, self.D.cpu().numpy())
        self.solver = DeviceSolver(
            self.dev, eps_tol=params.eps_tol, eps_inf=params.eps_inf, gamma_sys=gamma,
            tol_scale=ip.scale, tol_floor=ip.floor, diag_bound=diag_bound,
            adaptive=ip.adaptive, max_inner=ip.max_inner, halpern=params.halpern)
        self.checker = self.solver
        if self.checker_dev is not None:
            self.checker = DeviceSolver(
                self.checker_dev, eps_tol=params.eps_tol, eps_inf=params.eps_inf, gamma_sys=gamma,
                tol_scale=ip.scale, tol_floor=ip.floor, diag_bound=info.diag_bound,
                adaptive=ip.adaptive, max_inner=ip.max_inner, halpern=params.halpern)
        if group is not None:
            group.connect(self.solver)
        ph("solver_create")

    def read(self, which: int) -> np.ndarray:
        """A whole vector; a row shard joins the ranks' slices (collective)."""
        out = self.checker.read(which)
        return out if self.group is None else self.group.concat(out)

    def report(self, cr, need_slack: bool) -> ResidualReport:
        slack = self.read(DeviceSolver.DUAL_SLACK) if need_slack else None
        return certify.report_from_check(cr, self.con_scale, self.cost_inf, slack)

    # certification on the original problem (identity unless scaling is on)
    def check(self, with_rays: bool):
        if self.checker is self.solver:
            return self.solver.check(with_rays)
        self.checker.import_scaled(self.solver, self.D, self.E)
        cr = self.checker.check(with_rays)
        if with_rays:  # engine.py:443-453 on the iterating solver too: window restarts
            self.solver.reset_window()
            sc = self.solver.get_scalars()
            sc.block_len, sc.have_avg_prev = 0, 1
            self.solver.set_scalars(sc)
        return cr

    def mark_cert(self):
        if self.checker is not self.solver:
            self.checker.import_scaled(self.solver, self.D, self.E)
        self.checker.mark_cert()

    def forget_window(self):
        """After a halted window (engine.py:407-417): no previous averages."""
        if self.checker is not self.solver:
            sc = self.checker.get_scalars()
            sc.have_avg_prev, sc.block_len = 0, 0
            self.checker.set_scalars(sc)


def _scaled_diag_bound(quad, d: np.ndarray) -> float:
    """QuadOperator.diag_bound() of D Q D (inner.py:102) for the scaled solve."""
    d2 = d * d
    if quad.kind == "diagonal":
        return float((d2 * quad.values).max(initial=0.0))
    if quad.kind == "sparse":
        return float((d2 * quad.diag).max(initial=0.0))
    rsq = np.bincount(quad.r.indices, weights=quad.r.data ** 2, minlength=quad.n)
    return float((d2 * (quad.p.diag + rsq)).max(initial=0.0))


def solve(problem, params: Optional[SolverParams] = None, progress: Optional[ProgressCallback] = None,
          device: int = 0, monitor: Optional[Callable[[int, int], None]] = None, group=None,
          marks: Optional[Sequence[int]] = None, stats: Optional[dict] = None) -> SolveResult:
    """Run until optimality, an infeasibility certificate, or a limit
    (engine.py:339-498).  ``problem`` may be this package's QpProblem or the
    reference's (rebuilt field by field).

    ``monitor(outer, inner)`` (extension, not in the reference API) is called
    at every certification point right after the device check, with the
    cumulative outer and BB-inner iteration counts -- bench.py brackets
    certification windows with CUDA events from it.

    ``marks`` (extension): outer-iteration counts at which a window is split
    (without a certification point -- the device loop simply continues in the
    next graph launch, so the trajectory is unchanged); with ``marks`` given,
    ``monitor`` is called right after the window that reaches each mark
    instead of at certification points.  bench.py times outer iterations
    [W, W+K) with it, the same range its reference arm times.

    ``group`` (extension, shard.PeerGroup): solve this problem row-sharded
    with the group's other ranks; every rank calls solve
    with the same problem and params and gets the same result.

    ``stats`` (extension): a dict that receives branch counters of the loop --
    ``halts`` (device windows stopped by a non-finite move, the overflow
    rollback of engine.py:407-417) and ``rollbacks_divergence``
    (engine.py:484-487)."""
    params = params or SolverParams()
    ph = _Phases()
    counters = stats if stats is not None else {}
    counters.update(halts=0, rollbacks_divergence=0)
    problem = QpProblem.from_any(problem)
    validate_dims(problem)  # the data checks of validate() run on the device (_Run)
    ph("validate")
    start = time.monotonic()
    v0 = _StartVector(problem.n, params.norm_seed) if problem.constraint_matrix.nnz else None
    run = _Run(problem, params, progress, device, group, ph)
    sol = run.solver
    rs = _Round(omega=params.omega0, eta=0.0, theta=params.theta)
    rs.eta = estimate_eta(sol, problem, params, v0)
    ph("estimate_eta")
    tol0 = params.inner.initial if params.inner.adaptive else params.inner.fixed_tol
    sc = nat.Scalars()
    sc.eta, sc.omega, sc.theta, sc.inner_tol = rs.eta, rs.omega, rs.theta, tol0
    sol.init(sc)
    # host buffers of the result vectors, paged in while the loop runs
    run.checker.prefault((DeviceSolver.X_EVAL, DeviceSolver.Y, DeviceSolver.DUAL_SLACK))

    n_outer = n_inner = restarts = 0

    def finish(status, report, cert):
        ph("loop")
        x = run.read(DeviceSolver.X_EVAL)
        y = run.read(DeviceSolver.Y)
        if report.dual_slack is None:
            report = dataclasses.replace(report, dual_slack=run.read(DeviceSolver.DUAL_SLACK))
        ph("read_back")
        ph.dump()
        return SolveResult(status=status, x=x, y=y, report=report, certificate=cert,
                           outer_iterations=n_outer, inner_iterations=n_inner, restarts=restarts,
                           seconds=time.monotonic() - start)

    # sharded: reading the slack is collective, so every rank reads it
    want_slack = progress is not None or group is not None
    ph("init")
    cr = run.check(with_rays=False)
    report = run.report(cr, want_slack)
    ph("first_check")
    rs.best_residual_round_start = report.kkt_max
    rs.last_check_kkt = report.kkt_max
    if progress is not None:
        progress(0, report, rs.omega, rs.round)
    if certify.check_optimal(report, params.eps_tol):
        return finish(SolveStatus.OPTIMAL, report, None)
    run.mark_cert()
    best_kkt_seen = report.kkt_max
    stall_checks = 0
    probe_until = 0
    rp = params.restart
    check_every = params.check_every
    pending_marks = sorted({int(k) for k in marks if int(k) > 0}) if marks is not None else []

    def push(**kw):
        s = sol.get_scalars()
        for k, v in kw.items():
            setattr(s, k, v)
        sol.set_scalars(s)
        return s

    def rollback_round():
        # engine.py:303-319 (vectors on the device)
        sol.rollback()
        rs.round += 1
        rs.theta = rs.theta / 2.0 if rs.theta >= THETA_BACKOFF_FLOOR else 0.0
        rs.last_check_kkt = rs.best_residual_round_start
        push(k=0, theta=rs.theta)

    def reanchor(kkt):
        # engine.py:322-333 (and the vector half of _do_restart)
        sol.restart()
        rs.round += 1
        rs.best_residual_round_start = kkt
        rs.last_check_kkt = kkt

    while n_outer < params.iter_limit:
        probing = n_outer < probe_until
        sc = push(probing=int(probing))
        window = check_every - (n_outer % check_every)
        window = min(window, params.iter_limit - n_outer)
        if probing:
            window = min(window, probe_until - n_outer)
        elif rp.enabled:
            window = min(window, max(1, rp.max_round_len - sc.k))
        if pending_marks:
            window = min(window, pending_marks[0] - n_outer)
        sol.run(window)
        sc = sol.get_scalars()
        n_outer += sc.iters_done
        n_inner += sc.inner_sum
        while pending_marks and pending_marks[0] <= n_outer:
            if pending_marks.pop(0) == n_outer and monitor is not None:
                monitor(n_outer, n_inner)
        if sc.halted:
            # engine.py:407-417: overflow inside the round
            counters["halts"] += 1
            sol.rollback()
            rs.round += 1
            rs.theta = rs.theta / 2.0 if rs.theta >= THETA_BACKOFF_FLOOR else 0.0
            rs.last_check_kkt = rs.best_residual_round_start
            run.mark_cert()
            probe_until = 0
            sol.reset_window()
            run.forget_window()
            push(k=0, theta=rs.theta, halted=0, block_len=0, have_avg_prev=0)
            continue
        at_cap = (not probing) and rp.enabled and sc.k >= rp.max_round_len
        if not (n_outer % check_every == 0 or at_cap or n_outer == params.iter_limit):
            continue  # window ended at the probe boundary
        # ---- certification point (engine.py:436-494) -----------------------
        cr = run.check(with_rays=True)
        if monitor is not None and marks is None:
            monitor(n_outer, n_inner)
        report = run.report(cr, want_slack)
        kkt = report.kkt_max
        if progress is not None:
            progress(n_outer, report, rs.omega, rs.round)
        if certify.check_optimal(report, params.eps_tol):
            return finish(SolveStatus.OPTIMAL, report, None)
        order = (0, 1) if cr.have_avg_prev else (1,)
        for j in order:
            hit = certify.primal_ray_test(cr, j, params.eps_inf)
            if hit is not None:
                ray = run.read(DeviceSolver.YRAY0 + j)
                return finish(SolveStatus.PRIMAL_INFEASIBLE, report,
                              Certificate(CertificateKind.PRIMAL_RAY, ray, hit[0], hit[1]))
        for j in order:
            hit = certify.dual_ray_test(cr, j, params.eps_tol, params.eps_inf, run.gamma_sys)
            if hit is not None:
                ray = run.read(DeviceSolver.XRAY0 + j)
                return finish(SolveStatus.DUAL_INFEASIBLE, report,
                              Certificate(CertificateKind.DUAL_RAY, ray, hit[0], hit[1]))
        run.mark_cert()
        if math.isfinite(kkt) and kkt < STALL_IMPROVEMENT * best_kkt_seen:
            best_kkt_seen = min(best_kkt_seen, kkt)
            stall_checks = 0
        else:
            stall_checks += 1
        k_now = sol.get_scalars().k
        if probing:
            if n_outer >= probe_until:
                if stall_checks == 0:
                    reanchor(kkt)
                    push(k=0)
                else:
                    probe_until = n_outer + rp.max_round_len
        elif stall_checks >= STALL_CHECKS:
            probe_until = n_outer + rp.max_round_len
        elif not math.isfinite(kkt) or kkt > DIVERGENCE_FACTOR * rs.best_residual_round_start:
            counters["rollbacks_divergence"] += 1
            rollback_round()
            run.mark_cert()
        elif rp.enabled and restart_decision(k_now, rs, kkt, params):
            if kkt < rs.best_residual_round_start:  # anti-windup, engine.py:284-290
                rs.omega = pid_update(rs, math.sqrt(cr.pid_dx2), math.sqrt(cr.pid_dy2), params)
            reanchor(kkt)
            restarts += 1
            push(k=0, omega=rs.omega)
        else:
            rs.last_check_kkt = kkt
        if params.time_limit is not None:
            out_of_time = time.monotonic() - start >= params.time_limit
            if group is not None:  # a clock reading: every rank must take the same branch
                out_of_time = group.agree_any(out_of_time)
            if out_of_time:
                return finish(SolveStatus.TIME_LIMIT, report, None)

    cr = run.check(with_rays=False)
    return finish(SolveStatus.ITERATION_LIMIT, run.report(cr, False), None)
