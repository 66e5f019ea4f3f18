"""GPU: the row-sharded (multi-GPU) solve path, SURVEY.md §8(e).

Every test runs P virtual ranks on the one B200 of the test box
(shard.LocalGroup: one thread + CUDA stream per rank, peer stores are local
stores) -- the exact kernels, peer-store replication, mailbox exchanges and
graph barriers of a P-GPU run.  Contract as for one GPU (identical status,
objective within 1e-6, outer within +-10% of the reference golden), plus:
every rank returns bitwise-identical vectors and counts (all reductions are
combined in rank order on every rank).
"""

import numpy as np
import pytest

import instances
from conftest import golden
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import SolverParams, shard

pytestmark = pytest.mark.gpu


def run_sharded(p, prm, nranks):
    res = shard.solve_local(p, prm, nranks=nranks, timeout=600)
    r0 = res[0]
    for r in res[1:]:
        assert r.status == r0.status
        assert r.outer_iterations == r0.outer_iterations and r.inner_iterations == r0.inner_iterations
        assert np.array_equal(r.x, r0.x) and np.array_equal(r.y, r0.y)
        assert np.array_equal(r.report.dual_slack, r0.report.dual_slack)
    return r0


def check_golden(res, g):
    assert res.status.value == g["status"]
    assert abs(res.outer_iterations - g["outer"]) <= 0.10 * g["outer"]
    if g["status"] == "optimal":
        obj = g["objective"]
        assert abs(res.report.primal_objective - obj) <= 1e-6 * max(1.0, abs(obj))
        assert res.report.kkt_max <= g["eps_tol"]


@pytest.mark.parametrize("spec,fname,nranks", [
    ("c1:0", "ref_c1_s0.json", 2),
    ("c1:0", "ref_c1_s0.json", 8),
    ("rqp:300:150:sparse:0.05:7", "ref_rqp_300_150_sparse_0.05_7.json", 3),
    ("rqp:500:300:diagonal:0.02:5", "ref_rqp_500_300_diagonal_0.02_5.json", 4),
    ("c2:1e4:5e3:0", "ref_c2_1e4_5e3_0.json", 4),
    ("c5:5e4:500:0:diag", "ref_c5_5e4_500_0_diag.json", 2),
])
def test_sharded_matches_reference_golden(cuda, spec, fname, nranks):
    g = golden(fname)
    res = run_sharded(instances.build(spec), SolverParams(eps_tol=g["eps_tol"]), nranks)
    check_golden(res, g)
    if spec == "c1:0":  # the sharded trajectory reproduces the reference's counts exactly
        assert (res.outer_iterations, res.inner_iterations) == (g["outer"], g["inner"])


@pytest.mark.parametrize("spec,fname", [("c4u:1e3:1", "ref_c4u_1e3_1.json"), ("c4i:1e3:1", "ref_c4i_1e3_1.json")])
def test_sharded_infeasibility_certificates(cuda, spec, fname):
    g = golden(fname)
    p = instances.build(spec)
    res = run_sharded(p, SolverParams(eps_tol=g["eps_tol"]), 2)
    check_golden(res, g)
    single = aq.solve(p, SolverParams(eps_tol=g["eps_tol"]))
    assert res.certificate is not None and single.certificate is not None
    assert res.certificate.kind == single.certificate.kind
    # the ray is gathered whole from both shards
    np.testing.assert_allclose(res.certificate.ray, single.certificate.ray, rtol=1e-9, atol=1e-12)


def test_sharded_matches_single_gpu_trajectory(cuda):
    """Same instance, same iteration budget: the P-rank iterate equals the
    1-GPU iterate up to reduction-order rounding."""
    p = aq.random_qp(800, 500, "sparse", density=0.02, seed=11)
    prm = SolverParams(eps_tol=1e-12, iter_limit=256)
    one = aq.solve(p, prm)
    for nranks in (2, 5):
        sh = run_sharded(p, prm, nranks)
        assert sh.status == one.status == aq.SolveStatus.ITERATION_LIMIT
        np.testing.assert_allclose(sh.x, one.x, rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(sh.y, one.y, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("spec,fname,nranks", [
    ("rqp:300:150:low_rank:0.05:3", "ref_rqp_300_150_low_rank_0.05_3.json", 2),  # CSR R: R x all-reduced
    ("c3:2e3:100:0", "ref_c3_2e3_100_0.json", 2),                               # dense factor R (C3 twin)
    ("c3:2e4:100:0", "ref_c3_2e4_100_0.json", 3),
])
def test_sharded_low_rank_matches_reference_golden(cuda, spec, fname, nranks):
    """Low-rank Q = P + R'R row-sharded: R is split by columns, each rank's
    R x is a partial sum all-reduced (k values, rank order) before R'(R x)."""
    g = golden(fname)
    res = run_sharded(instances.build(spec), SolverParams(eps_tol=g["eps_tol"]), nranks)
    check_golden(res, g)


def test_sharded_sparse_c5_twin(cuda):
    """The sparse-Q C5 twin (banded A, Q band i +- 1000) over 4 ranks."""
    g = golden("ref_c5_5e4_500_0.json")
    res = run_sharded(instances.build("c5:5e4:500:0"), SolverParams(eps_tol=g["eps_tol"]), 4)
    check_golden(res, g)


@pytest.mark.parametrize("spec", ["c5:5e4:500:0", "c5:5e4:500:0:diag", "c3:2e4:100:0"])
def test_storage_shrinks_with_ranks(cuda, spec):
    """Storage shards: a rank's persistent problem memory and solver workspace
    are ~1/P of the whole problem's (instances too large
    for one GPU)."""
    from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver

    p = instances.build(spec)
    ctx = DeviceContext.get(0)

    def solver_bytes(dev):
        import ctypes as C

        sz = C.c_size_t()
        ctx.lib.aqp_solver_sizes(dev.handle, C.byref(sz))
        return sz.value

    whole = DeviceProblem(p, ctx)
    w_prob, w_sol = whole.persistent_bytes, solver_bytes(whole)
    whole.close()
    P = 4
    plans = shard.plan(p, P)
    for r in range(P):
        dev = DeviceProblem(p, ctx, part=shard.local_part(p, plans, r))
        assert dev.persistent_bytes <= 1.2 * w_prob / P + (1 << 20), (r, dev.persistent_bytes, w_prob)
        assert solver_bytes(dev) <= 1.3 * w_sol / P + (8 << 20), (r, solver_bytes(dev), w_sol)
        dev.close()
