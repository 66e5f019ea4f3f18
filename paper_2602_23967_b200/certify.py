"""KKT residual report, certificates, and the host half of the tests.

The device computes the raw reductions of a certification point
(``aqp_check_result`` in include/aqp.h); this module restates the formulas
of the reference (``anchorqp/certify.py:63-164``) on those numbers -- same
operation order and Python float semantics -- so every comparison the
solve loop makes (optimality, ray tests, restarts) is the reference's.
"""

from __future__ import annotations

import dataclasses
import enum
import math

import numpy as np

from .model import Bounds


class CertificateKind(str, enum.Enum):
    """PRIMAL_RAY certifies primal infeasibility (a y-ray); DUAL_RAY certifies
    dual infeasibility / unboundedness (an x-ray)."""

    PRIMAL_RAY = "primal_ray"
    DUAL_RAY = "dual_ray"


@dataclasses.dataclass(frozen=True)
class Certificate:
    kind: CertificateKind
    ray: np.ndarray
    violation: float
    improvement: float


@dataclasses.dataclass(frozen=True)
class ResidualReport:
    r_primal: float
    r_dual: float
    r_gap: float
    primal_objective: float
    dual_objective: float
    dual_slack: np.ndarray

    @property
    def kkt_max(self) -> float:
        return max(self.r_primal, self.r_dual, self.r_gap)


# certify.py:106 -- absolute guard on the inf-normalised ray
ABS_RAY_GUARD = 1e-10


def finite_bound_scale(bounds: Bounds) -> float:
    """max |finite bound| over both sides (reference certify.py:54-60); setup scalar."""
    scale = 0.0
    for arr in (bounds.lower, bounds.upper):
        fin = arr[np.isfinite(arr)]
        if fin.size:
            scale = max(scale, float(np.abs(fin).max()))
    return scale


def linf(v: np.ndarray) -> float:
    return float(np.abs(v).max()) if len(v) else 0.0


def _support(pos: float, neg: float, bad: int) -> float:
    # model.py:57-71: +inf on a bad side, else upper.z+ + lower.z-
    return float("inf") if bad else pos + neg


def report_from_check(cr, con_scale: float, cost_inf: float, dual_slack: np.ndarray) -> ResidualReport:
    """certify.py:63-95 evaluated on device reductions."""
    r_primal = cr.primal_viol / (1.0 + con_scale)
    r_dual = cr.dual_viol / (1.0 + max(cr.qx_inf, cr.aty_inf, cost_inf))
    p_r = _support(cr.pr_pos, cr.pr_neg, cr.pr_bad)
    p_y = _support(cr.py_pos, cr.py_neg, cr.py_bad)
    xqx, cx = cr.xqx, cr.cx
    gap_num = abs(xqx + cx + p_r + p_y)
    gap_den = 1.0 + max(abs(0.5 * xqx + cx), abs(0.5 * xqx + p_r + p_y))
    r_gap = gap_num / gap_den
    return ResidualReport(
        r_primal=r_primal,
        r_dual=r_dual,
        r_gap=r_gap,
        primal_objective=0.5 * xqx + cx,
        dual_objective=-p_r - 0.5 * xqx - p_y,
        dual_slack=dual_slack,
    )


def check_optimal(report: ResidualReport, eps_tol: float) -> bool:
    """certify.py:98-100."""
    return report.kkt_max <= eps_tol


def primal_ray_test(cr, j: int, eps_inf: float):
    """certify.py:109-133 on candidate j; returns (violation, improvement) or None."""
    norm = cr.yr_norm[j]
    if norm == 0.0 or not math.isfinite(norm):
        return None
    violation = cr.yr_viol[j]
    b_value = (_support(cr.yr_var_pos[j], cr.yr_var_neg[j], cr.yr_var_bad[j])
               + _support(cr.yr_con_pos[j], cr.yr_con_neg[j], cr.yr_con_bad[j]))
    if not math.isfinite(b_value) or b_value >= 0.0:
        return None
    b_minus = -b_value
    if violation <= eps_inf * b_minus and violation <= ABS_RAY_GUARD * (1.0 + cr.yr_aty_inf[j]):
        return violation, b_minus
    return None


def dual_ray_test(cr, j: int, eps_tol: float, eps_inf: float, gamma_sys: float):
    """certify.py:136-164 on candidate j; returns (violation, improvement) or None."""
    norm = cr.xr_norm[j]
    if norm == 0.0 or not math.isfinite(norm):
        return None
    improvement = cr.xr_improvement[j]
    if not improvement < -eps_tol:
        return None
    violation = max(cr.xr_viol_x[j], cr.xr_viol_s[j], cr.xr_qd_inf[j] / gamma_sys)
    if violation <= eps_inf:
        return violation, improvement
    return None


def default_gamma_sys(problem) -> float:
    """1 + row-norm bound of Q (certify.py:167-169); setup scalar."""
    return 1.0 + problem.quad.inf_norm_bound()
