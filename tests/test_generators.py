"""Instance generators: the reference generators are restated draw for draw
(hashes recorded from the reference itself), and the scale generators build
well-formed, feasible-by-construction instances deterministically."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_2602_23967_b200 import generators as g
from paper_2602_23967_b200 import validate


def digest(p):
    h = hashlib.sha256()
    q = p.quad
    arrs = [p.cost, p.constraint_matrix.indptr, p.constraint_matrix.indices, p.constraint_matrix.data,
            p.var_bounds.lower, p.var_bounds.upper, p.con_bounds.lower, p.con_bounds.upper]
    if q.kind == "diagonal":
        arrs.append(q.values)
    elif q.kind == "sparse":
        arrs += [q.upper.indptr, q.upper.indices, q.upper.data, q.diag]
    else:
        arrs += [q.p.upper.indptr, q.p.upper.indices, q.p.upper.data, q.p.diag, q.r.indptr, q.r.indices, q.r.data]
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


H = golden("generator_hashes.json")


@pytest.mark.parametrize("args", [(2000, 1000, "sparse", 0.01, 0), (40, 20, "diagonal", 0.3, 1),
                                  (30, 15, "low_rank", 0.3, 4), (300, 150, "sparse", 0.05, 7)])
def test_random_qp_identical_to_reference(args):
    assert digest(g.random_qp(*args)) == H["random_qp" + repr(args)]


def test_lasso_identical_to_reference():
    a, b = g.random_lasso_data(30, 20, density=0.3, seed=2)
    assert digest(g.make_lasso_qp(a, b)) == H["make_lasso_qp(random_lasso_data(30,20,0.3,2))"]


def _csr_ok(a):
    assert a.indptr[0] == 0 and a.indptr[-1] == a.nnz
    for i in range(min(a.rows, 50)):
        seg = a.indices[a.indptr[i]:a.indptr[i + 1]]
        assert np.all(np.diff(seg) > 0)


def test_lasso_style_c2_shape():
    p = g.lasso_style_qp(20_000, 10_000, seed=3)
    validate(p)
    assert (p.n, p.m) == (20_000, 10_000)
    _csr_ok(p.constraint_matrix)
    assert 7.9 * p.m <= p.constraint_matrix.nnz <= 8 * p.m
    q = p.quad.to_scipy()
    assert abs(q - q.T).max() == 0
    # strict diagonal dominance => positive definite
    off = np.asarray(abs(q).sum(axis=1)).ravel() - q.diagonal()
    assert np.all(q.diagonal() > off)
    assert digest(p) == digest(g.lasso_style_qp(20_000, 10_000, seed=3))


def test_portfolio_c3_shape():
    p = g.portfolio_qp(3000, 10, sectors=5, seed=1)
    validate(p)
    assert p.m == 6 and p.constraint_matrix.nnz == 2 * p.n
    assert p.quad.r.rows == 10 and p.quad.r.nnz == 10 * 3000
    assert np.all(p.var_bounds.lower == 0) and np.allclose(p.var_bounds.upper, 20 / 3000)


def test_infeasible_pair_c4_shape():
    unb, inf = g.infeasible_pair(2000, seed=1)
    validate(unb)
    validate(inf)
    a0 = unb.constraint_matrix.to_scipy().tocsc()
    assert a0[:, 0].nnz == 0 and unb.cost[0] == -1.0 and unb.quad.values[0] == 0.0
    assert inf.m == unb.m + 2
    last = inf.constraint_matrix.to_scipy()[-2:].toarray()
    assert np.array_equal(last[0], last[1]) and (inf.con_bounds.lower[-2:] == [1.0, 2.0]).all()


def test_banded_c5_locality():
    p = g.banded_qp(10_000, half_width=50, seed=0)
    validate(p)
    a = p.constraint_matrix
    rows = np.repeat(np.arange(a.rows), np.diff(a.indptr))
    assert np.abs(a.indices - rows).max() <= 50
    assert p.quad.to_scipy().nnz <= 10_000 + 2 * (2 * 10_000)
