"""GPU: the solve entry's setup work on the device (aqp_problem_setup_info,
aqp_h2d / aqp_d2h) against the host restatements of the reference.

* validate()'s data checks (reference model.py:168-206): every violation kind
  raises, through solve(), the same error class and message as the host
  ``validate`` -- including which violation wins when several are present;
* inf_norm_bound / default_gamma_sys (linalg.py:218-220, 260-263,
  certify.py:167-169), diag_bound, finite_bound_scale and |c|_inf are
  BITWISE the numpy values (sequential row / column sums in bincount order);
* a row shard's per-rank structs combine to the whole problem's;
* the staged copies round-trip bytes exactly.
"""

import dataclasses

import numpy as np
import pytest

import instances
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import Bounds, DiagonalQuad, SparseMatrix, certify, shard
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem
from paper_2602_23967_b200.engine import _setup_info
from paper_2602_23967_b200.errors import InvalidProblem
from paper_2602_23967_b200.linalg import SparseLowRankQuad, SparseQuad
from paper_2602_23967_b200.model import validate

pytestmark = pytest.mark.gpu

SPECS = ["c1:0", "rqp:300:150:sparse:0.05:7", "rqp:500:300:diagonal:0.02:5", "rqp:300:150:low_rank:0.05:3",
         "c3:2e3:100:0", "c2:1e4:5e3:0", "c5:5e4:500:0", "c5:5e4:500:0:diag", "c4u:1e3:1", "c4i:1e3:1"]


def host_scalars(p):
    return dict(gamma=certify.default_gamma_sys(p), con_scale=certify.finite_bound_scale(p.con_bounds),
                cost_inf=certify.linf(p.cost), diag_bound=p.quad.diag_bound())


def device_scalars(info, p):
    qb = info.q_bound
    if p.quad.kind == "sparse_low_rank":
        qb = qb + info.r_one * info.r_inf
    return dict(gamma=1.0 + qb, con_scale=info.con_scale, cost_inf=info.cost_inf, diag_bound=info.diag_bound)


@pytest.mark.parametrize("spec", SPECS)
def test_setup_scalars_bitwise(cuda, spec):
    p = instances.build(spec)
    dev = DeviceProblem(p, DeviceContext.get(0))
    info = dev.setup_info()
    assert device_scalars(info, p) == host_scalars(p)  # exact float equality
    assert (info.var_nan, info.var_wrong_inf, info.con_nan, info.con_wrong_inf) == (0, 0, 0, 0)
    assert info.var_first_inverted == info.con_first_inverted == -1
    assert (info.cost_nonfinite, info.a_nonfinite, info.q_nonfinite) == (0, 0, 0)



def test_setup_scalars_explicit_diag_and_missing_diagonal(cuda):
    """SparseQuad with an explicit diag argument that differs from the stored
    diagonal, and an upper triangle that stores only some diagonals (no split
    diagonal on the device)."""
    rng = np.random.default_rng(5)
    n = 700
    dense = np.triu(rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.01))
    keep = rng.random(n) < 0.5
    dense[np.arange(n), np.arange(n)] = np.where(keep, rng.random(n) + 0.1, 0.0)
    upper = SparseMatrix.from_dense(dense)
    base = aq.random_qp(n, 300, "sparse", density=0.02, seed=2)
    for diag in (None, rng.random(n) * 3.0):
        p = dataclasses.replace(base, quad=SparseQuad(upper, diag))
        info = DeviceProblem(p, DeviceContext.get(0)).setup_info()
        assert device_scalars(info, p) == host_scalars(p)


@pytest.mark.parametrize("spec,nranks", [("c1:0", 3), ("c5:5e4:500:0", 4), ("c3:2e3:100:0", 2),
                                         ("rqp:300:150:low_rank:0.05:3", 2), ("rqp:500:300:diagonal:0.02:5", 3)])
def test_setup_scalars_sharded_combine(cuda, spec, nranks):
    p = instances.build(spec)
    plans = shard.plan(p, nranks)
    groups = shard.LocalGroup.create(nranks)
    ctx = DeviceContext.get(0)
    devs = [DeviceProblem(p, ctx, part=shard.local_part(p, plans, r)) for r in range(nranks)]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(nranks) as ex:
        infos = list(ex.map(lambda r: _setup_info(devs[r], p, groups[r]), range(nranks)))
    for info in infos:
        assert device_scalars(info, p) == host_scalars(p)


def _bad_variants(p):
    """(name, problem) pairs with one or more data violations."""
    n, m = p.n, p.m
    lo, hi = p.var_bounds.lower.copy(), p.var_bounds.upper.copy()
    clo, chi = p.con_bounds.lower.copy(), p.con_bounds.upper.copy()
    a = p.constraint_matrix
    out = []

    def vb(l, h):
        return dataclasses.replace(p, var_bounds=Bounds(l, h))

    def cb(l, h):
        return dataclasses.replace(p, con_bounds=Bounds(l, h))

    l2 = lo.copy(); l2[7] = np.nan; out.append(("var_nan", vb(l2, hi)))
    l2 = lo.copy(); l2[3] = np.inf; out.append(("var_wrong_inf", vb(l2, hi)))
    l2, h2 = lo.copy(), hi.copy(); l2[11], h2[11] = 2.0, 1.0; l2[5], h2[5] = 4.0, 3.0
    out.append(("var_inverted_first", vb(l2, h2)))
    c2 = chi.copy(); c2[2] = -np.inf; out.append(("con_wrong_inf", cb(clo, c2)))
    c1, c2 = clo.copy(), chi.copy(); c1[m - 1], c2[m - 1] = 1.0, -1.0; out.append(("con_inverted", cb(c1, c2)))
    c = p.cost.copy(); c[n - 1] = np.inf; out.append(("cost", dataclasses.replace(p, cost=c)))
    d = a.data.copy(); d[a.nnz // 2] = np.inf  # SparseMatrix itself rejects NaN
    out.append(("a_inf", dataclasses.replace(p, constraint_matrix=SparseMatrix(a.rows, a.cols, a.indptr, a.indices, d))))
    q = p.quad
    qd = q.upper.data.copy(); qd[len(qd) // 3] = -np.inf
    out.append(("q_inf", dataclasses.replace(p, quad=SparseQuad(SparseMatrix(n, n, q.upper.indptr, q.upper.indices, qd), q.diag))))
    # several at once: the first in validate()'s order wins
    c = p.cost.copy(); c[0] = np.nan
    c1, c2 = clo.copy(), chi.copy(); c1[4], c2[4] = 5.0, 0.0
    out.append(("con_inverted_and_cost", dataclasses.replace(p, cost=c, con_bounds=Bounds(c1, c2))))
    return out


@pytest.mark.parametrize("idx", range(9))
def test_device_validation_matches_host(cuda, idx):
    p = aq.random_qp(60, 40, "sparse", density=0.1, seed=4)
    name, bad = _bad_variants(p)[idx]
    with pytest.raises(InvalidProblem) as host:
        validate(bad)
    with pytest.raises(InvalidProblem) as dev:
        aq.solve(bad)
    assert type(dev.value) is type(host.value), name
    assert str(dev.value) == str(host.value), name


@pytest.mark.parametrize("kind", ["diagonal", "low_rank"])
def test_device_validation_quad_kinds(cuda, kind):
    p = aq.random_qp(50, 30, kind, density=0.1, seed=9)
    if kind == "diagonal":
        v = p.quad.values.copy(); v[3] = np.nan
        bad = dataclasses.replace(p, quad=DiagonalQuad(v))
    else:
        r = p.quad.r
        d = r.data.copy(); d[1] = np.inf
        bad = dataclasses.replace(p, quad=SparseLowRankQuad(p.quad.p, SparseMatrix(r.rows, r.cols, r.indptr, r.indices, d)))
    with pytest.raises(InvalidProblem) as host:
        validate(bad)
    with pytest.raises(InvalidProblem) as dev:
        aq.solve(bad)
    assert type(dev.value) is type(host.value) and str(dev.value) == str(host.value)


@pytest.mark.parametrize("nbytes", [0, 1000, (8 << 20) + 13, (100 << 20) + 8])
def test_staged_copies_round_trip(cuda, nbytes):
    import ctypes as C

    ctx = DeviceContext.get(0)
    src = np.random.default_rng(nbytes).integers(0, 256, nbytes, dtype=np.uint8)
    t = ctx.upload(src)
    assert t.numel() == max(nbytes, 1)
    back = np.empty(nbytes, dtype=np.uint8)
    from paper_2602_23967_b200 import _native as nat

    nat.check(ctx.lib.aqp_d2h(ctx.handle, C.c_void_p(back.ctypes.data), C.c_void_p(t.data_ptr()), nbytes))
    assert np.array_equal(back, src)
    if nbytes:
        assert np.array_equal(t[:nbytes].cpu().numpy(), src)
