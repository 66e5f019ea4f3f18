"""GPU: the solve entry point against the oracle and the reference's golden runs.

Contract (BASELINE.json north_star): identical status; objective and KKT
within 1e-6 relative at the 1e-8 tolerance; outer iterations within +-10%.
On config 1 and the C4 families the device trajectory reproduces the
reference's to the last count, which the exact-count assertions record.
"""

import math

import numpy as np
import pytest

import instances
import oracle
from conftest import golden
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import (
    Bounds,
    DiagonalQuad,
    QpProblem,
    RestartParams,
    SolverParams,
    SolveStatus,
    SparseMatrix,
    random_qp,
    solve,
)
from paper_2602_23967_b200.errors import InvertedBound

pytestmark = pytest.mark.gpu
INF = np.inf


def assert_parity(res, status, outer, objective, eps=1e-8):
    assert res.status.value == status
    assert abs(res.outer_iterations - outer) <= 0.10 * outer
    if status == "optimal":
        assert res.report.kkt_max <= eps
        assert abs(res.report.primal_objective - objective) <= 1e-6 * max(1.0, abs(objective))


GOLDENS = [
    ("c1:0", "ref_c1_s0.json"), ("c1:1", "ref_c1_s1.json"), ("c1:2", "ref_c1_s2.json"),
    ("c1:3", "ref_c1_s3.json"), ("c1:4", "ref_c1_s4.json"),
    ("c4u:1e3:1", "ref_c4u_1e3_1.json"), ("c4i:1e3:1", "ref_c4i_1e3_1.json"),
    ("c4ur:1e3:1", "ref_c4ur_1e3_1.json"), ("c4ir:1e3:1", "ref_c4ir_1e3_1.json"),
    ("c4ur:1e4:1", "ref_c4ur_1e4_1.json"), ("c4ir:1e4:1", "ref_c4ir_1e4_1.json"),
    ("c4u:1e4:1", "ref_c4u_1e4_1.json"), ("c4i:1e4:1", "ref_c4i_1e4_1.json"),
    ("c4u:1e5:1", "ref_c4u_1e5_1.json"), ("c4i:1e5:1", "ref_c4i_1e5_1.json"),
    ("c2:1e4:5e3:0", "ref_c2_1e4_5e3_0.json"),
    ("c3:2e3:100:0", "ref_c3_2e3_100_0.json"), ("c3:2e4:100:0", "ref_c3_2e4_100_0.json"),
    ("c5:5e4:500:0", "ref_c5_5e4_500_0.json"), ("c5:5e4:500:0:diag", "ref_c5_5e4_500_0_diag.json"),
    ("c5:5e5:500:0", "ref_c5_5e5_500_0.json"),  # C5/100 (reference: 674 s on one core)
    # a real QPS file (ranges, free rows, negative UP, FX/MI/PL, QMATRIX) read by
    # this repo's reader; the golden is the reference solving its own parse
    ("qps:tests/golden/qps_mixed_400.qps", "ref_qps_mixed_400.json"),
    ("rqp:300:150:sparse:0.05:7", "ref_rqp_300_150_sparse_0.05_7.json"),
    ("rqp:300:150:low_rank:0.05:3", "ref_rqp_300_150_low_rank_0.05_3.json"),
    ("rqp:500:300:diagonal:0.02:5", "ref_rqp_500_300_diagonal_0.02_5.json"),
]


@pytest.mark.parametrize("spec,fname", GOLDENS)
def test_matches_reference_golden_run(cuda, spec, fname):
    g = golden(fname)
    res = solve(instances.build(spec), SolverParams(eps_tol=g["eps_tol"]))
    assert_parity(res, g["status"], g["outer"], g["objective"], g["eps_tol"])
    if g["status"] != "optimal":
        assert res.certificate is not None
    assert abs(res.inner_iterations - g["inner"]) <= 0.10 * max(g["inner"], 10)
    if spec.startswith(("c1:", "c4", "c2:1e4")):
        # on config 1, the C4 families and the C2 twin the device trajectory is
        # the reference's trajectory to the last count (longer runs drift in the
        # last bits of the reduction order, inside the +-10% contract)
        assert (res.outer_iterations, res.inner_iterations, res.restarts) == (g["outer"], g["inner"], g["restarts"])


SUITE = [(n, m, kind, seed) for kind in ("sparse", "diagonal", "low_rank") for (n, m, seed) in
         [(8, 5, 1), (15, 9, 2), (25, 12, 3), (30, 15, 4), (12, 20, 5), (40, 10, 6), (20, 20, 7)]]


@pytest.mark.parametrize("n,m,kind,seed", SUITE)
def test_random_suite_against_oracle(cuda, n, m, kind, seed):
    """Like the reference's 40-instance suite (tests/test_testkit.py:65-74)."""
    p = random_qp(n, m, kind, seed=seed)
    prm = SolverParams(eps_tol=1e-8)
    ref = oracle.solve(p, prm)
    res = solve(p, prm)
    assert_parity(res, ref["status"], ref["outer"], ref["report"]["primal_objective"])
    assert abs(res.inner_iterations - ref["inner"]) <= 0.10 * max(ref["inner"], 10)


# ---------------------------------------------------------------- reference TestSolve (tests/test_engine.py:251-331)
def test_simple_qp(cuda):
    p = QpProblem(quad=DiagonalQuad(np.ones(1)), cost=np.array([-1.0]),
                  constraint_matrix=SparseMatrix.from_coo(0, 1, [], [], []),
                  var_bounds=Bounds(np.array([0.0]), np.array([10.0])), con_bounds=Bounds(np.zeros(0), np.zeros(0)))
    res = solve(p, SolverParams(eps_tol=1e-8))
    assert res.status is SolveStatus.OPTIMAL
    assert abs(res.x[0] - 1.0) <= 1e-6


def test_primal_infeasible_detected(cuda):
    p = QpProblem(quad=DiagonalQuad(np.zeros(1)), cost=np.zeros(1), constraint_matrix=SparseMatrix.from_dense([[1.0]]),
                  var_bounds=Bounds(np.array([0.0]), np.array([INF])),
                  con_bounds=Bounds(np.array([-INF]), np.array([-1.0])))
    res = solve(p, SolverParams(iter_limit=50_000))
    ref = oracle.solve(p, SolverParams(iter_limit=50_000))
    assert res.status is SolveStatus.PRIMAL_INFEASIBLE and ref["status"] == "primal_infeasible"
    assert res.certificate is not None and res.outer_iterations == ref["outer"]
    assert np.array_equal(res.certificate.ray, ref["certificate"][1])


def test_dual_infeasible_detected(cuda):
    p = QpProblem(quad=DiagonalQuad(np.zeros(1)), cost=np.array([-1.0]),
                  constraint_matrix=SparseMatrix.from_coo(0, 1, [], [], []),
                  var_bounds=Bounds(np.array([0.0]), np.array([INF])), con_bounds=Bounds(np.zeros(0), np.zeros(0)))
    res = solve(p, SolverParams(iter_limit=50_000))
    assert res.status is SolveStatus.DUAL_INFEASIBLE
    assert res.certificate is not None and res.certificate.improvement < 0


def test_iteration_limit(cuda):
    res = solve(random_qp(8, 5, "sparse", seed=3), SolverParams(eps_tol=1e-12, iter_limit=10))
    assert res.status is SolveStatus.ITERATION_LIMIT and res.outer_iterations == 10


def test_invalid_problem_raises(cuda):
    p = QpProblem(quad=DiagonalQuad(np.zeros(1)), cost=np.zeros(1), constraint_matrix=SparseMatrix.from_dense([[1.0]]),
                  var_bounds=Bounds(np.array([1.0]), np.array([0.0])),
                  con_bounds=Bounds(np.array([0.0]), np.array([1.0])))
    with pytest.raises(InvertedBound):
        solve(p)


def test_deterministic_bitwise(cuda):
    p = random_qp(10, 6, "sparse", seed=11)
    a, b = solve(p, SolverParams(eps_tol=1e-7)), solve(p, SolverParams(eps_tol=1e-7))
    assert a.status == b.status and a.outer_iterations == b.outer_iterations
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)


def test_deterministic_bitwise_large(cuda):
    p = instances.build("c2:2e5:1e5:1")
    prm = SolverParams(eps_tol=1e-12, iter_limit=300)
    a, b = solve(p, prm), solve(p, prm)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and a.inner_iterations == b.inner_iterations


def test_progress_callback_cadence(cuda):
    seen = []
    solve(random_qp(6, 4, "diagonal", seed=5), SolverParams(eps_tol=1e-30, iter_limit=300, check_every=64),
          progress=lambda it, rep, omega, rnd: seen.append((it, rep.dual_slack.shape)))
    assert seen[0][0] == 0 and all(it % 64 == 0 for it, _ in seen[:-1])
    assert seen[0][1] == (6,)


def test_time_limit(cuda):
    res = solve(random_qp(20, 10, "sparse", seed=2), SolverParams(eps_tol=1e-30, time_limit=0.2, iter_limit=10 ** 9))
    assert res.status is SolveStatus.TIME_LIMIT and res.seconds >= 0.2


def test_zero_constraint_matrix(cuda):
    # eta = 1e8 when A has no nonzeros (reference tests/test_engine.py:88-96)
    p = QpProblem(quad=DiagonalQuad(np.array([2.0])), cost=np.array([-4.0]),
                  constraint_matrix=SparseMatrix.from_coo(1, 1, [], [], []), var_bounds=Bounds.free(1),
                  con_bounds=Bounds(np.array([-INF]), np.array([INF])))
    res = solve(p, SolverParams(eps_tol=1e-9))
    ref = oracle.solve(p, SolverParams(eps_tol=1e-9))
    assert res.status.value == ref["status"] and res.outer_iterations == ref["outer"]
    assert res.x[0] == pytest.approx(2.0, abs=1e-6)


# ---------------------------------------------------------------- reference TestReductions (tests/test_engine.py:334-370)
def _fixture_lp():
    return QpProblem(quad=DiagonalQuad(np.zeros(3)), cost=np.array([-1.0, 0.5, 0.25]),
                     constraint_matrix=SparseMatrix.from_dense([[2.0, 0.0, 0.0], [0.0, 2.0, 0.0]]),
                     var_bounds=Bounds(np.zeros(3), np.full(3, 2.0)),
                     con_bounds=Bounds(np.array([-1.0, 0.5]), np.array([1.0, 1.5])))


def _hand_pdhg(problem, eta, steps, anchor):
    lo, hi = problem.var_bounds.lower, problem.var_bounds.upper
    lc, uc = problem.con_bounds.lower, problem.con_bounds.upper
    a = problem.constraint_matrix.to_scipy().toarray()
    x, y = np.clip(np.zeros(problem.n), lo, hi), np.zeros(problem.m)
    ax0, ay0 = x.copy(), y.copy()
    out = []
    for k in range(steps):
        xp = np.clip(x - eta * (problem.cost + a.T @ y), lo, hi)
        w = y / eta + a @ (2.0 * xp - x)
        yp = eta * (w - np.clip(w, lc, uc))
        if anchor:
            x = (k + 1.0) / (k + 2.0) * xp + 1.0 / (k + 2.0) * ax0
            y = (k + 1.0) / (k + 2.0) * yp + 1.0 / (k + 2.0) * ay0
        else:
            x, y = xp, yp
        out.append((x.copy(), y.copy()))
    return out


@pytest.mark.parametrize("anchor", [True, False])
def test_matches_hand_rolled_pdhg_over_50_steps(cuda, anchor):
    p = _fixture_lp()

    def prm(k):
        return SolverParams(theta=0.0, pid_gains=(0.0, 0.0, 0.0), restart=RestartParams(enabled=False),
                            eps_tol=1e-30, halpern=anchor, iter_limit=k)

    ref = _hand_pdhg(p, 0.998 / 2.0, 50, anchor)
    for k in (1, 2, 3, 5, 13, 34, 50):
        res = solve(p, prm(k))
        assert np.abs(res.x - ref[k - 1][0]).max() <= 1e-12
        assert np.abs(res.y - ref[k - 1][1]).max() <= 1e-12


def test_reflected_halpern_against_oracle(cuda):
    p = random_qp(30, 15, "sparse", seed=9)
    prm = SolverParams(eps_tol=1e-8, theta=0.5)
    ref = oracle.solve(p, prm)
    res = solve(p, prm)
    assert_parity(res, ref["status"], ref["outer"], ref["report"]["primal_objective"])


# ---------------------------------------------------------------- full-size properties (BASELINE sizes)
@pytest.mark.slow
def test_config2_full_size_converges(cuda):
    """C2 at n=1e6, m=5e5 to 1e-8: optimal, KKT below tolerance, and the
    reported objective agrees with the primal objective recomputed from x."""
    p = instances.build("c2:1e6:5e5:0")
    res = solve(p, SolverParams(eps_tol=1e-8))
    assert res.status is SolveStatus.OPTIMAL and res.report.kkt_max <= 1e-8
    x = res.x
    assert np.all(x >= p.var_bounds.lower) and np.all(x <= p.var_bounds.upper)
    qx = p.quad.to_scipy() @ x
    obj = 0.5 * float(x @ qx) + float(p.cost @ x)
    assert obj == pytest.approx(res.report.primal_objective, rel=1e-9)
    try:
        g = golden("ref_c2_1e6_5e5_0.json")
    except FileNotFoundError:
        return
    if g["status"] == "optimal":
        assert_parity(res, g["status"], g["outer"], g["objective"])


@pytest.mark.slow
def test_config4_full_size_pair(cuda):
    unb, inf = (instances.build(s) for s in ("c4u:1e5:1", "c4i:1e5:1"))
    ru, ri = solve(unb, SolverParams(eps_tol=1e-8)), solve(inf, SolverParams(eps_tol=1e-8))
    assert ru.status is SolveStatus.DUAL_INFEASIBLE and ri.status is SolveStatus.PRIMAL_INFEASIBLE
    for name, r in (("c4u_1e5_1", ru), ("c4i_1e5_1", ri)):
        try:
            g = golden(f"ref_{name}.json")
        except FileNotFoundError:
            continue
        assert_parity(r, g["status"], g["outer"], g["objective"])


@pytest.mark.parametrize("scaling", ["ruiz", "ruiz_pc"])
@pytest.mark.parametrize("spec,fname", [("c1:0", "ref_c1_s0.json"),
                                        ("rqp:300:150:low_rank:0.05:3", "ref_rqp_300_150_low_rank_0.05_3.json"),
                                        ("rqp:500:300:diagonal:0.02:5", "ref_rqp_500_300_diagonal_0.02_5.json"),
                                        ("c4i:1e3:1", "ref_c4i_1e3_1.json"), ("c4u:1e3:1", "ref_c4u_1e3_1.json")])
def test_opt_in_scaling_keeps_status_and_objective(cuda, spec, fname, scaling):
    """SolverParams(scaling=...) (extension, off by default): device-side
    Ruiz / Pock-Chambolle equilibration; certification stays on the original
    problem, so status and objective match the reference (iteration counts
    differ by design)."""
    g = golden(fname)
    res = solve(instances.build(spec), SolverParams(eps_tol=g["eps_tol"], scaling=scaling))
    assert res.status.value == g["status"]
    if g["status"] == "optimal":
        assert res.report.kkt_max <= g["eps_tol"]
        assert abs(res.report.primal_objective - g["objective"]) <= 1e-6 * max(1.0, abs(g["objective"]))
    else:
        assert res.certificate is not None


@pytest.mark.parametrize("fname", ["ref_rb_theta0.9_rqp_300_150_sparse_0.05_7.json",
                                   "ref_rb_theta0.99_rqp_300_150_sparse_0.05_7.json",
                                   "ref_rb_eta1000_rqp_300_150_sparse_0.05_7.json"])
def test_rollback_branches_match_reference(cuda, fname):
    """The two rollback branches of the reference loop, forced by parameters
    and recorded from the reference with per-branch call counts
    (oracle/run_reference.py): a large Halpern reflection theta diverges and
    is rolled back to the round anchor with theta halved (engine.py:484-487,
    303-319) until it converges; a 1000x step scale overflows inside the
    device window (the device halt flag, engine.py:407-417) and diverges at
    checks, until the iteration limit."""
    g = golden(fname)
    prm = SolverParams(eps_tol=g["eps_tol"], iter_limit=g["iter_limit"], **g["params"])
    stats = {}
    trace = []
    res = solve(instances.build(g["spec"]), prm, stats=stats,
                progress=lambda it, rep, om, rnd: trace.append((it, rnd)))
    ref_rb = g["rollbacks"]
    assert res.status.value == g["status"]
    assert stats["halts"] == ref_rb["overflow"] and stats["rollbacks_divergence"] == ref_rb["divergence"]
    assert (stats["halts"] > 0) == (ref_rb["overflow"] > 0)  # the device halt flag fired iff the reference overflowed
    if g["status"] == "optimal":
        assert_parity(res, g["status"], g["outer"], g["objective"], g["eps_tol"])
        assert res.restarts == g["restarts"]
    else:
        assert res.outer_iterations == g["outer"]
    # the round counter at every certification point follows the reference's
    assert [r for _, r in trace] == [t[5] for t in g["trace"]]

