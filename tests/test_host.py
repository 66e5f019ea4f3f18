"""Host-side logic (no device): parameter validation, data model, the
tolerance / restart / PID rules, and the residual and certificate formulas
that the host evaluates on device reductions -- each checked against the
oracle restatement of the reference (or the reference's hand examples)."""

import math

import numpy as np
import pytest

import oracle
from paper_2602_23967_b200 import (
    Bounds,
    DiagonalQuad,
    QpProblem,
    RestartParams,
    SolverParams,
    SparseMatrix,
    SparseQuad,
    cone_of,
    random_qp,
    validate,
)
from paper_2602_23967_b200 import _native as nat
from paper_2602_23967_b200 import certify, engine
from paper_2602_23967_b200.errors import DimensionMismatch, InvertedBound, NonFiniteData

INF = np.inf


# ---------------------------------------------------------------- params (reference tests/test_engine.py:395-)
def test_solver_params_validation():
    for kw in (dict(eps_tol=0.0), dict(theta=1.0), dict(omega0=0.0), dict(iter_limit=0), dict(time_limit=-1.0)):
        with pytest.raises(ValueError):
            SolverParams(**kw)
    with pytest.raises(ValueError):
        RestartParams(beta_sufficient=0.9, beta_necessary=0.5)
    RestartParams(enabled=False, beta_sufficient=0.9, beta_necessary=0.5)


# ---------------------------------------------------------------- model (reference tests/test_model.py)
@pytest.mark.parametrize("lo,hi,dual_y,dual_r,recc", [
    (-INF, INF, 0, 0, 3), (-INF, 1.0, 1, 2, 2), (0.0, INF, 2, 1, 1), (0.0, 1.0, 3, 3, 0)])
def test_cone_tables(lo, hi, dual_y, dual_r, recc):
    b = Bounds(np.array([lo]), np.array([hi]))
    assert cone_of(b, "dual_y")[0] == dual_y
    assert cone_of(b, "dual_r")[0] == dual_r
    assert cone_of(b, "recession")[0] == recc
    with pytest.raises(ValueError):
        cone_of(b, "bogus")


def _prob(**over):
    base = dict(quad=DiagonalQuad(np.zeros(1)), cost=np.zeros(1), constraint_matrix=SparseMatrix.from_dense([[1.0]]),
                var_bounds=Bounds(np.array([0.0]), np.array([1.0])), con_bounds=Bounds(np.array([0.0]), np.array([1.0])))
    base.update(over)
    return QpProblem(**base)


def test_validate_errors():
    validate(_prob())
    with pytest.raises(InvertedBound):
        validate(_prob(var_bounds=Bounds(np.array([1.0]), np.array([0.0]))))
    with pytest.raises(DimensionMismatch):
        validate(_prob(cost=np.zeros(2)))
    with pytest.raises(NonFiniteData):
        validate(_prob(cost=np.array([np.nan])))
    with pytest.raises(NonFiniteData):
        validate(_prob(con_bounds=Bounds(np.array([np.inf]), np.array([np.inf]))))


def test_sparse_matrix_contract():
    a = SparseMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [2.0, 3.0, 1.0])
    assert a.nnz == 2 and np.array_equal(a.to_scipy().toarray(), [[0, 5], [1, 0]])
    with pytest.raises(NonFiniteData):
        SparseMatrix.from_dense(np.array([[np.nan]]))
    with pytest.raises(DimensionMismatch):
        SparseMatrix(1, 2, [0, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        DiagonalQuad(np.array([-1.0]))
    with pytest.raises(ValueError):
        SparseQuad.from_symmetric(np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_reference_objects_are_adopted():
    p = random_qp(12, 7, "low_rank", seed=2)
    again = QpProblem.from_any(p)
    assert again is p
    class Duck:  # a reference-shaped object with foreign classes
        pass
    d = Duck()
    d.quad, d.cost, d.constraint_matrix = p.quad, p.cost, p.constraint_matrix
    d.var_bounds, d.con_bounds, d.name = p.var_bounds, p.con_bounds, "duck"
    q = QpProblem.from_any(d)
    assert q.n == p.n and q.quad.kind == "sparse_low_rank"


# ---------------------------------------------------------------- rules (reference tests/test_inner.py:127-152, test_engine.py:187-248)
def _round(base, last):
    return engine._Round(omega=1.0, eta=1.0, theta=0.0, best_residual_round_start=base, last_check_kkt=last)


def test_restart_rule():
    p = SolverParams()
    assert engine.restart_decision(10, _round(1.0, 0.5), 0.1, p)
    assert engine.restart_decision(p.restart.max_round_len, _round(1.0, 0.9), 0.9, p)
    assert not engine.restart_decision(10, _round(1.0, 0.95), 0.9, p)
    assert engine.restart_decision(10, _round(1.0, 0.5), 0.6, p)


def test_pid_rule():
    rs = _round(1.0, 1.0)
    w = engine.pid_update(rs, 2.0, 1.0, SolverParams(pid_gains=(0.5, 0.0, 0.0)))
    assert math.log(w) == pytest.approx(-0.5 * math.log(2.0))
    rs = _round(1.0, 1.0)
    engine.pid_update(rs, 2.0, 1.0, SolverParams())
    assert rs.pid_last_error == pytest.approx(math.log(2.0))
    rs = _round(1.0, 1.0)
    rs.omega = 3.0
    assert engine.pid_update(rs, 0.0, 1.0, SolverParams()) == 3.0
    rs = _round(1.0, 1.0)
    rs.omega = 1e-6
    for _ in range(50):
        rs.omega = engine.pid_update(rs, 1e-12, 1e3, SolverParams(pid_gains=(5.0, 0.0, 0.0)))
        assert 1e-6 <= rs.omega <= 1e6


# ---------------------------------------------------------------- formulas on device reductions
def _fake_check(inst, x, y):
    """CheckResult filled with the reductions the device computes, evaluated
    in numpy from their definitions."""
    cr = nat.CheckResult()
    ax, qx, aty = inst.ax(x), inst.qx(x), inst.aty(y)
    r = qx + inst.c + aty
    rp = oracle.cone_project(r, inst.cone_r)
    cr.primal_viol = oracle.linf(ax - np.clip(ax, inst.clo, inst.chi))
    cr.dual_viol = oracle.linf(r - rp)
    cr.qx_inf, cr.aty_inf = oracle.linf(qx), oracle.linf(aty)

    def parts(z, lo, hi):
        pos, neg = z > 0, z < 0
        bad = int(np.any(pos & np.isinf(hi)) or np.any(neg & np.isinf(lo)))
        return float(hi[pos & np.isfinite(hi)] @ z[pos & np.isfinite(hi)]), float(lo[neg & np.isfinite(lo)] @ z[neg & np.isfinite(lo)]), bad

    cr.pr_pos, cr.pr_neg, cr.pr_bad = parts(-rp, inst.vlo, inst.vhi)
    cr.py_pos, cr.py_neg, cr.py_bad = parts(oracle.cone_project(y, inst.cone_y), inst.clo, inst.chi)
    cr.xqx, cr.cx = float(x @ qx), float(inst.c @ x)
    return cr


@pytest.mark.parametrize("kind,seed", [("sparse", 1), ("diagonal", 2), ("low_rank", 3)])
def test_report_formulas_match_oracle(kind, seed):
    p = random_qp(25, 12, kind, seed=seed)
    inst = oracle.Instance(p)
    rng = np.random.default_rng(seed)
    x = oracle.clamp(rng.standard_normal(25), inst.vlo, inst.vhi)
    y = oracle.cone_project(rng.standard_normal(12), inst.cone_y)
    ref = oracle.residuals(inst, x, y)
    cr = _fake_check(inst, x, y)
    rep = certify.report_from_check(cr, certify.finite_bound_scale(p.con_bounds), certify.linf(p.cost), None)
    assert rep.r_primal == pytest.approx(ref["r_primal"], rel=1e-12, abs=0)
    assert rep.r_dual == pytest.approx(ref["r_dual"], rel=1e-12)
    assert rep.r_gap == pytest.approx(ref["r_gap"], rel=1e-9)
    assert rep.primal_objective == pytest.approx(ref["primal_objective"], rel=1e-12)


def test_primal_ray_formula_hand_example():
    # reference tests/test_certify.py:128-133: x in [0, inf), x <= -1  ->  y-ray fires
    p = QpProblem(quad=DiagonalQuad(np.zeros(1)), cost=np.zeros(1), constraint_matrix=SparseMatrix.from_dense([[1.0]]),
                  var_bounds=Bounds(np.array([0.0]), np.array([INF])), con_bounds=Bounds(np.array([-INF]), np.array([-1.0])))
    inst = oracle.Instance(p)
    ref = oracle.primal_ray(inst, np.array([1.0]), 1e-9)
    cr = nat.CheckResult()
    ray = oracle.cone_project(np.array([1.0]), inst.cone_y)
    cr.yr_norm[1] = oracle.linf(ray)
    at = inst.aty(ray / cr.yr_norm[1])
    atp = oracle.cone_project(at, inst.cone_r)
    cr.yr_viol[1], cr.yr_aty_inf[1] = oracle.linf(at - atp), oracle.linf(at)
    cr.yr_var_pos[1], cr.yr_var_neg[1], cr.yr_var_bad[1] = 0.0, 0.0, 0
    cr.yr_con_pos[1], cr.yr_con_neg[1], cr.yr_con_bad[1] = -1.0, 0.0, 0
    hit = certify.primal_ray_test(cr, 1, 1e-9)
    assert ref is not None and hit is not None
    assert hit == (ref[2], ref[3]) == (0.0, 1.0)


def test_dual_ray_formula_rejects_non_descent():
    cr = nat.CheckResult()
    cr.xr_norm[1], cr.xr_improvement[1] = 1.0, -1e-7
    assert certify.dual_ray_test(cr, 1, 1e-6, 1e-9, 1.0) is None
    cr.xr_improvement[1] = -1.0
    assert certify.dual_ray_test(cr, 1, 1e-6, 1e-9, 1.0) == (0.0, -1.0)
    cr.xr_qd_inf[1] = 1e-6
    assert certify.dual_ray_test(cr, 1, 1e-6, 1e-9, 2.0) is None
