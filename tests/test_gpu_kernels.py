"""GPU: the registry kernels through the C ABI (include/aqp.h "registry" section)
against the reference's recorded outputs (bitwise) and against dense algebra
(the reference's own tolerances, tests/test_kernels.py / test_linalg.py)."""

import os

import numpy as np
import pytest
import scipy.sparse as sp
from numpy.testing import assert_allclose

import oracle
from conftest import GOLDEN
from paper_2602_23967_b200 import (
    DiagonalQuad,
    SparseLowRankQuad,
    SparseMatrix,
    SparseQuad,
    ZeroMatrix,
    estimate_norm,
    quad_apply,
)
from paper_2602_23967_b200 import kernels as kern

pytestmark = pytest.mark.gpu
K = np.load(os.path.join(GOLDEN, "kernels.npz"))


@pytest.mark.parametrize("t", range(5))
def test_csr_products_bitwise_reference(cuda, t):
    ip, ix, dv = K[f"mv{t}_indptr"], K[f"mv{t}_indices"], K[f"mv{t}_data"]
    rows, cols = len(ip) - 1, len(K[f"mv{t}_x"])
    assert np.array_equal(kern.csr_matvec(ip, ix, dv, K[f"mv{t}_x"], rows), K[f"mv{t}_ax"])
    assert np.array_equal(kern.csr_matvec_t(ip, ix, dv, K[f"mv{t}_y"], cols), K[f"mv{t}_aty"])


@pytest.mark.parametrize("t", range(4))
def test_sym_product_bitwise_reference(cuda, t):
    out = kern.sym_matvec(K[f"sym{t}_indptr"], K[f"sym{t}_indices"], K[f"sym{t}_data"], K[f"sym{t}_diag"],
                          K[f"sym{t}_x"])
    assert np.array_equal(out, K[f"sym{t}_out"])


def test_vector_kernels_reference(cuda):
    x, g, q, lin, lo, hi = (K[k] for k in ("v_x", "v_g", "v_q", "v_lin", "v_lo", "v_hi"))
    assert np.array_equal(kern.clamp(x, lo, hi), K["k_clamp"])
    assert np.array_equal(kern.cone_project(x, K["v_codes"]), K["k_cone"])
    assert np.array_equal(kern.diag_prox_step(x, q, lin, 0.37, lo, hi), K["k_prox"])
    assert np.array_equal(kern.dual_step(x, g, 1.7, lo, hi), K["k_dual"])
    assert np.array_equal(kern.lincomb3(0.3, x, 0.6, g, -0.25, lin), K["k_lin3"])
    assert np.array_equal(kern.axpby(2.0, x, -1.0, g), K["k_axpby"])
    # reductions: fixed tree order, not the Cython sequential order
    assert kern.natural_res_sq(x, g, lo, hi) == pytest.approx(K["k_natres"][0], rel=1e-13)
    z = x * (np.isfinite(lo) & np.isfinite(hi))
    assert kern.support_p(z, lo, hi) == pytest.approx(K["k_support"][0], rel=1e-13)
    assert kern.support_p(np.array([1.0]), np.array([0.0]), np.array([np.inf])) == np.inf
    assert kern.support_p(np.array([0.0]), np.array([-np.inf]), np.array([np.inf])) == 0.0


def _random_csr(rng, rows, cols, density=0.4):
    m = sp.random(rows, cols, density=density, random_state=rng).tocsr()
    m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data, m.toarray()


def test_csr_matvec_matches_dense(cuda, rng):
    # reference tests/test_kernels.py:39-46
    for _ in range(10):
        rows, cols = rng.integers(1, 20, size=2)
        ip, ix, dv, dense = _random_csr(rng, rows, cols)
        x = rng.standard_normal(cols)
        assert_allclose(kern.csr_matvec(ip, ix, dv, x, rows), dense @ x, atol=1e-14)
        y = rng.standard_normal(rows)
        assert_allclose(kern.csr_matvec_t(ip, ix, dv, y, cols), dense.T @ y, atol=1e-14)


@pytest.mark.parametrize("rows,cols,dens", [(200_000, 150_000, 5e-5), (40, 300_000, 0.5), (3, 2_000_000, 0.9)])
def test_csr_large_and_long_rows_match_oracle(cuda, rng, rows, cols, dens):
    """Short rows (thread/warp tiles) and rows split across many blocks (long
    segments) against the sequential oracle."""
    m = sp.random(rows, cols, density=dens, random_state=rng, format="csr")
    m.sort_indices()
    ip, ix = m.indptr.astype(np.int64), m.indices.astype(np.int64)
    x, y = rng.standard_normal(cols), rng.standard_normal(rows)
    a, b = kern.csr_matvec(ip, ix, m.data, x, rows), oracle.csr_matvec(ip, ix, m.data, x, rows)
    assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max())
    at, bt = kern.csr_matvec_t(ip, ix, m.data, y, cols), oracle.csr_matvec_t(ip, ix, m.data, y, cols)
    assert np.array_equal(at, bt)


def test_sym_matvec_matches_dense(cuda, rng):
    # reference tests/test_kernels.py:49-64
    for _ in range(10):
        n = int(rng.integers(1, 20))
        base = rng.standard_normal((n, n))
        full = base + base.T
        up = sp.triu(sp.csr_matrix(full)).tocsr()
        up.sort_indices()
        x = rng.standard_normal(n)
        out = kern.sym_matvec(up.indptr.astype(np.int64), up.indices.astype(np.int64), up.data, np.diag(full).copy(), x)
        assert_allclose(out, full @ x, atol=1e-12)


def _random_quad(rng, n, kind):
    if kind == "diagonal":
        q = rng.uniform(0, 2, n)
        return DiagonalQuad(q), np.diag(q)
    f = rng.standard_normal((n, max(1, n // 2)))
    psd = f @ f.T
    if kind == "sparse":
        return SparseQuad.from_symmetric(psd), psd
    r = rng.standard_normal((3, n)) * (rng.random((3, n)) < 0.6)
    return SparseLowRankQuad(SparseQuad.from_symmetric(psd), SparseMatrix.from_dense(r)), psd + r.T @ r


def test_quad_apply_matches_dense(cuda, rng):
    # reference tests/test_linalg.py:80-88
    for kind in ("diagonal", "sparse", "low_rank"):
        for _ in range(6):
            n = int(rng.integers(1, 50))
            quad, dense = _random_quad(rng, n, kind)
            x = rng.standard_normal(n)
            ref = dense @ x
            assert np.abs(quad_apply(quad, x) - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_estimate_norm_contract(cuda, rng):
    # reference tests/test_linalg.py:115-145
    assert estimate_norm(SparseMatrix.from_dense(np.eye(2))) == pytest.approx(1.0, abs=1e-6)
    assert estimate_norm(SparseMatrix.from_dense(np.diag([3.0, 1.0]))) == pytest.approx(3.0, abs=1e-4)
    with pytest.raises(ZeroMatrix):
        estimate_norm(SparseMatrix.from_dense(np.zeros((1, 2))))
    for _ in range(5):
        dense = rng.standard_normal((6, 9))
        est, true = estimate_norm(SparseMatrix.from_dense(dense)), np.linalg.norm(dense, 2)
        assert 0.99 * true <= est <= true * (1 + 1e-12)
    dense = rng.standard_normal((4, 6))
    a = estimate_norm(SparseMatrix.from_dense(dense))
    assert abs(a - estimate_norm(SparseMatrix.from_dense(np.vstack([dense, np.zeros((3, 6))])))) <= 1e-8
    a = SparseMatrix.from_dense(rng.standard_normal((5, 5)))
    assert estimate_norm(a, seed=7) == estimate_norm(a, seed=7)


def test_estimate_norm_matches_oracle(cuda):
    import instances

    p = instances.build("c1:0")
    ours = estimate_norm(p.constraint_matrix, 100, 0)
    ref = oracle.estimate_norm(oracle.Instance(p), 100, 0)
    assert ours == pytest.approx(ref, rel=1e-13)
