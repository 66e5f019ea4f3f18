"""Seeded synthetic instances for the BASELINE configs (harness input only).

* ``random_qp`` / ``make_lasso_qp`` / ``random_lasso_data`` restate the
  reference generators (``anchorqp/generators.py:22-152``) draw for draw, so
  ``random_qp(2000, 1000, "sparse", density=0.01, seed=0)`` is bit-identical
  to the reference's config-1 instance (checked in ``tests/test_generators.py``
  against committed hashes).
* ``lasso_style_qp`` (C2), ``portfolio_qp`` (C3), ``infeasible_pair`` (C4)
  and ``banded_qp`` (C5) are the scale-capable generators SURVEY.md §8(d)
  specifies: they build CSR arrays directly (no dense FF', which is what
  makes ``random_qp`` unusable past n ~ 1e4) and return ordinary
  ``QpProblem`` objects that the CPU reference can consume unchanged.

All generators run on the host: they create input data, they are not part of
the solve path.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .errors import DimensionMismatch
from .linalg import DiagonalQuad, SparseLowRankQuad, SparseMatrix, SparseQuad
from .model import Bounds, QpProblem

STRUCTURES = ("diagonal", "sparse", "low_rank")


# ---------------------------------------------------------------------------
# reference generators (same RNG call sequence as anchorqp/generators.py)
# ---------------------------------------------------------------------------
def _uniform_sparse(rng, rows, cols, density):
    # anchorqp/generators.py:13-17
    return sp.random(rows, cols, density=density, random_state=rng,
                     data_rvs=lambda size: rng.uniform(-1.0, 1.0, size))


def _csr_rowdot(a: SparseMatrix, x: np.ndarray) -> np.ndarray:
    # row-sequential sum from 0.0, the order of the reference's csr_matvec
    # (anchorqp/_kernels/_core.pyx:29-42); scipy's csr_matvec uses it too.
    return a.to_scipy() @ x


def random_qp(n: int, m: int, structure: str = "sparse", density: float = 0.3,
              seed: int = 0, rank: int = None) -> QpProblem:
    """Random feasible QP (anchorqp/generators.py:22-91)."""
    if n < 1 or m < 1:
        raise ValueError("n and m must be at least 1")
    if structure not in STRUCTURES:
        raise ValueError(f"structure must be one of {STRUCTURES}")
    if not 0.0 < density <= 1.0:
        raise ValueError("density must lie in (0, 1]")
    rng = np.random.default_rng(seed)

    boxed_only = np.zeros(n, dtype=bool)
    if structure == "diagonal":
        q = rng.uniform(0.05, 2.0, n)
        boxed_only = rng.random(n) < 0.2
        q[boxed_only] = 0.0
        quad = DiagonalQuad(q)
    elif structure == "sparse":
        f = _uniform_sparse(rng, n, n, density)
        qm = (f @ f.T).tocsr() + sp.diags(rng.uniform(0.05, 0.5, n))
        quad = SparseQuad.from_symmetric(qm)
    else:
        k = rank if rank is not None else max(1, min(5, n // 2))
        f = _uniform_sparse(rng, n, n, density)
        pm = (f @ f.T).tocsr() + sp.diags(rng.uniform(0.05, 0.5, n))
        rm = _uniform_sparse(rng, k, n, density)
        quad = SparseLowRankQuad(SparseQuad.from_symmetric(pm), SparseMatrix.from_scipy(rm))

    mid = rng.normal(0.0, 1.0, n)
    lower = mid - rng.uniform(0.2, 2.0, n)
    upper = mid + rng.uniform(0.2, 2.0, n)
    u = rng.random(n)
    lower_only = ~boxed_only & (u < 0.15)
    upper_only = ~boxed_only & (u >= 0.15) & (u < 0.30)
    free = ~boxed_only & (u >= 0.30) & (u < 0.40)
    lower[upper_only | free] = -np.inf
    upper[lower_only | free] = np.inf

    x0 = np.minimum(np.maximum(rng.normal(mid, 0.5), lower), upper)
    a = SparseMatrix.from_scipy(_uniform_sparse(rng, m, n, density))
    s0 = _csr_rowdot(a, x0)
    kind = rng.random(m)
    gap_lo = rng.uniform(0.1, 1.5, m)
    gap_hi = rng.uniform(0.1, 1.5, m)
    c_lo = np.where(kind < 0.2, s0, np.where(kind < 0.45, -np.inf, s0 - gap_lo))
    c_hi = np.where(kind < 0.2, s0, np.where((kind >= 0.45) & (kind < 0.70), np.inf, s0 + gap_hi))
    cost = rng.normal(0.0, 1.0, n)
    return QpProblem(quad=quad, cost=cost, constraint_matrix=a,
                     var_bounds=Bounds(lower, upper), con_bounds=Bounds(c_lo, c_hi),
                     name=f"random-{structure}-n{n}-m{m}-s{seed}")


def make_lasso_qp(a, b, lam: float = 0.0) -> QpProblem:
    """QP form of min |Ax-b|^2 + lam|x|_1 (anchorqp/generators.py:94-143)."""
    a_sp = a.to_scipy() if isinstance(a, SparseMatrix) else sp.csr_matrix(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a_sp.shape
    if b.shape != (m,):
        raise DimensionMismatch(f"b has shape {b.shape}, expected ({m},)")
    if lam == 0.0:
        lam = 0.01 * float(np.abs(a_sp.T @ b).max(initial=0.0))
        if lam <= 0.0:
            raise ValueError("default lambda rule degenerates; pass lam explicitly")
    if lam < 0.0:
        raise ValueError("lam must be positive")
    i_n = sp.eye(n, format="csr")
    i_m = sp.eye(m, format="csr")
    big = sp.bmat([[a_sp, None, -i_m], [i_n, -i_n, None], [-i_n, -i_n, None]], format="csr")
    quad = DiagonalQuad(np.concatenate([np.zeros(2 * n), 2.0 * np.ones(m)]))
    cost = np.concatenate([np.zeros(n), lam * np.ones(n), np.zeros(m)])
    vb = Bounds(np.concatenate([np.full(n, -np.inf), np.zeros(n), np.full(m, -np.inf)]),
                np.full(2 * n + m, np.inf))
    cb = Bounds(np.concatenate([b, np.full(2 * n, -np.inf)]), np.concatenate([b, np.zeros(2 * n)]))
    return QpProblem(quad=quad, cost=cost, constraint_matrix=SparseMatrix.from_scipy(big),
                     var_bounds=vb, con_bounds=cb, name="lasso")


def random_lasso_data(m: int, n: int, density: float = 0.5, seed: int = 0):
    """(A, b) with b = A x_sparse + noise (anchorqp/generators.py:146-152)."""
    rng = np.random.default_rng(seed)
    a_mat = _uniform_sparse(rng, m, n, density).tocsr()
    x_true = np.where(rng.random(n) < 0.2, rng.normal(0.0, 2.0, n), 0.0)
    b = a_mat @ x_true + 0.01 * rng.normal(0.0, 1.0, m)
    return SparseMatrix.from_scipy(a_mat), b


# ---------------------------------------------------------------------------
# scale-capable generators
# ---------------------------------------------------------------------------
def _csr_from_rows(rows: int, cols: int, col_ids: np.ndarray, vals: np.ndarray) -> SparseMatrix:
    """Canonical CSR from a (rows x k) block of column ids / values
    (duplicates within a row summed, columns sorted)."""
    k = col_ids.shape[1]
    r = np.repeat(np.arange(rows, dtype=np.int64), k)
    coo = sp.coo_matrix((vals.ravel(), (r, col_ids.ravel())), shape=(rows, cols))
    return SparseMatrix.from_scipy(coo)


def _row_pattern_bounds(rng, x0, pattern):
    """Variable box around a feasible x0: 30% upper-only, 30% lower-only,
    40% boxed with total width in [0.2, 2]."""
    n = len(x0)
    below = rng.uniform(0.1, 1.0, n)
    above = rng.uniform(0.1, 1.0, n)
    lower = x0 - below
    upper = x0 + above
    lower[pattern < 0.3] = -np.inf
    upper[(pattern >= 0.3) & (pattern < 0.6)] = np.inf
    return Bounds(lower, upper)


def _row_bounds(rng, s0):
    """Constraint rows around s0 = A x0: 30% equality, 30% <=, 20% ranged, 20% >=."""
    m = len(s0)
    kind = rng.random(m)
    gap_lo = rng.uniform(0.1, 1.0, m)
    gap_hi = rng.uniform(0.1, 1.0, m)
    lo = np.where(kind < 0.3, s0, np.where(kind < 0.6, -np.inf, s0 - gap_lo))
    hi = np.where(kind < 0.3, s0, np.where(kind < 0.8, s0 + gap_hi, np.inf))
    return Bounds(lo, hi)


def _dominant_sym(rng, n, pair_i, pair_j, pair_v) -> SparseQuad:
    """Q = D + S, S symmetric from upper pairs, D_ii = sum_j |S_ij| + U(0.05,1)
    (strictly diagonally dominant, hence positive definite)."""
    keep = pair_i != pair_j
    lo = np.minimum(pair_i, pair_j)[keep]
    hi = np.maximum(pair_i, pair_j)[keep]
    v = pair_v[keep]
    off = sp.coo_matrix((v, (lo, hi)), shape=(n, n)).tocsr()
    off.sum_duplicates()
    absrow = np.asarray(abs(off).sum(axis=1)).ravel() + np.asarray(abs(off).sum(axis=0)).ravel()
    d = absrow + rng.uniform(0.05, 1.0, n)
    upper = (off + sp.diags(d, format="csr")).tocsr()
    upper.sort_indices()
    return SparseQuad(SparseMatrix.from_scipy(upper))


def lasso_style_qp(n: int = 1_000_000, m: int = 500_000, seed: int = 0,
                   a_per_row: int = 8, q_pairs_per_row: int = 2) -> QpProblem:
    """C2: Lasso-style sparse QP, Q = D + S (~4 off-diagonals per row), A with
    ``a_per_row`` uniform columns per row, a feasible x0 embedded."""
    rng = np.random.default_rng(seed)
    npairs = q_pairs_per_row * n
    pi = rng.integers(0, n, npairs)
    pj = rng.integers(0, n, npairs)
    pv = rng.uniform(-1.0, 1.0, npairs)
    quad = _dominant_sym(rng, n, pi, pj, pv)
    cols = rng.integers(0, n, (m, a_per_row))
    vals = rng.uniform(-1.0, 1.0, (m, a_per_row))
    a = _csr_from_rows(m, n, cols, vals)
    x0 = rng.normal(0.0, 1.0, n)
    vb = _row_pattern_bounds(rng, x0, rng.random(n))
    cb = _row_bounds(rng, _csr_rowdot(a, x0))
    cost = rng.normal(0.0, 1.0, n)
    return QpProblem(quad=quad, cost=cost, constraint_matrix=a, var_bounds=vb, con_bounds=cb,
                     name=f"lasso-style-n{n}-m{m}-s{seed}")


def portfolio_qp(n: int = 5_000_000, k: int = 100, sectors: int = 20, seed: int = 0) -> QpProblem:
    """C3: factor-model portfolio, Q = diag(D) + F F' as SparseLowRankQuad(P=D, R=F')."""
    rng = np.random.default_rng(seed)
    f_t = rng.normal(0.0, np.sqrt(0.09 / k), (k, n))
    d = rng.uniform(0.01, 0.1, n)
    mu = rng.normal(0.05, 0.02, n)
    sector = rng.integers(0, sectors, n)
    p = SparseQuad(SparseMatrix(n, n, np.arange(n + 1), np.arange(n), d))
    r = SparseMatrix(k, n, np.arange(k + 1, dtype=np.int64) * n, np.tile(np.arange(n), k), f_t.ravel())
    # rows: budget 1'x = 1, then one "<= 0.2" row per sector
    order = np.argsort(sector, kind="stable")
    counts = np.bincount(sector, minlength=sectors)
    indptr = np.concatenate([[0, n], n + np.cumsum(counts)]).astype(np.int64)
    indices = np.concatenate([np.arange(n), order])
    # within a sector row the column ids must ascend: argsort(stable) gives that
    a = SparseMatrix(sectors + 1, n, indptr, indices, np.ones(2 * n))
    cb = Bounds(np.concatenate([[1.0], np.full(sectors, -np.inf)]),
                np.concatenate([[1.0], np.full(sectors, 0.2)]))
    vb = Bounds(np.zeros(n), np.full(n, 20.0 / n))
    return QpProblem(quad=SparseLowRankQuad(p, r), cost=-mu, constraint_matrix=a,
                     var_bounds=vb, con_bounds=cb, name=f"portfolio-n{n}-k{k}-s{seed}")


def diagonal_base_qp(n: int, m: int, seed: int = 1, per_row: int = 8) -> QpProblem:
    """Well-conditioned diagonal-Q base: q ~ U(0.5, 2) (strictly convex), A with
    ``per_row`` uniform columns per row, feasible x0 and the C2 bound patterns."""
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, (m, per_row))
    vals = rng.uniform(-1.0, 1.0, (m, per_row))
    a = _csr_from_rows(m, n, cols, vals)
    x0 = rng.normal(0.0, 1.0, n)
    vb = _row_pattern_bounds(rng, x0, rng.random(n))
    cb = _row_bounds(rng, _csr_rowdot(a, x0))
    return QpProblem(quad=DiagonalQuad(rng.uniform(0.5, 2.0, n)), cost=rng.normal(0.0, 1.0, n), constraint_matrix=a,
                     var_bounds=vb, con_bounds=cb, name=f"diag-base-n{n}-m{m}-s{seed}")


def infeasible_pair(n: int = 100_000, seed: int = 1, base: str = "diagonal"):
    """C4: (dual-unbounded, primal-infeasible) pair on one diagonal-Q base.

    ``base="diagonal"`` (default) uses :func:`diagonal_base_qp` (n, n/2): it
    certifies in ~1e3-5e4 outer iterations at n = 1e5.  ``base="random_qp"``
    is SURVEY.md §8(d)'s recipe ``random_qp(n, n//2, "diagonal", 10/n)``,
    whose zero-curvature coordinates delay certification past 1e6 iterations
    at n = 1e5 (on the reference and here alike).

    * unbounded: variable 0 gets q=0, c=-1, box [0, inf) and an empty column in A;
    * infeasible: one random 10-nnz row appended twice with equality targets 1 and 2.
    """
    if base == "random_qp":
        base = random_qp(n, max(1, n // 2), "diagonal", density=min(1.0, 10.0 / n), seed=seed)
    else:
        base = diagonal_base_qp(n, max(1, n // 2), seed=seed)
    a = base.constraint_matrix
    # --- dual-unbounded -----------------------------------------------------
    q = base.quad.values.copy()
    q[0] = 0.0
    c = base.cost.copy()
    c[0] = -1.0
    lo = base.var_bounds.lower.copy()
    hi = base.var_bounds.upper.copy()
    lo[0], hi[0] = 0.0, np.inf
    a_sp = a.to_scipy().tocoo()
    keep = a_sp.col != 0
    a0 = sp.csr_matrix((a_sp.data[keep], (a_sp.row[keep], a_sp.col[keep])), shape=a_sp.shape)
    unbounded = QpProblem(quad=DiagonalQuad(q), cost=c, constraint_matrix=SparseMatrix.from_scipy(a0),
                          var_bounds=Bounds(lo, hi), con_bounds=base.con_bounds,
                          name=f"dual-unbounded-n{n}-s{seed}")
    # --- primal-infeasible --------------------------------------------------
    rng = np.random.default_rng(seed + 7919)
    cols = np.sort(rng.choice(n, size=min(10, n), replace=False))
    vals = rng.uniform(-1.0, 1.0, len(cols))
    extra = sp.csr_matrix((np.concatenate([vals, vals]),
                           (np.repeat([0, 1], len(cols)), np.concatenate([cols, cols]))), shape=(2, n))
    a1 = sp.vstack([a.to_scipy(), extra], format="csr")
    cl = np.concatenate([base.con_bounds.lower, [1.0, 2.0]])
    cu = np.concatenate([base.con_bounds.upper, [1.0, 2.0]])
    infeasible = QpProblem(quad=base.quad, cost=base.cost, constraint_matrix=SparseMatrix.from_scipy(a1),
                           var_bounds=base.var_bounds, con_bounds=Bounds(cl, cu),
                           name=f"primal-infeasible-n{n}-s{seed}")
    return unbounded, infeasible


def banded_qp(n: int, m: int = None, half_width: int = 5000, seed: int = 0, per_row: int = 10,
              diagonal_q: bool = False) -> QpProblem:
    """C5: banded-local sparse QP.  Row i of A has ``per_row`` columns drawn from
    clip(i*n/m + U{-w..w}); Q = D + S with upper off-diagonals at (i, i+1) and
    (i, i+1000) (or a diagonal Q when ``diagonal_q``)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    centre = (np.arange(m, dtype=np.int64) * n) // m
    cols = np.clip(centre[:, None] + rng.integers(-half_width, half_width + 1, (m, per_row)), 0, n - 1)
    vals = rng.uniform(-1.0, 1.0, (m, per_row))
    a = _csr_from_rows(m, n, cols, vals)
    if diagonal_q:
        quad = DiagonalQuad(rng.uniform(0.05, 1.0, n))
    else:
        far = min(1000, max(1, n - 1))
        i1 = np.arange(n - 1, dtype=np.int64)
        i2 = np.arange(max(0, n - far), dtype=np.int64)
        pi = np.concatenate([i1, i2])
        pj = np.concatenate([i1 + 1, i2 + far])
        pv = rng.uniform(-1.0, 1.0, len(pi))
        quad = _dominant_sym(rng, n, pi, pj, pv)
    x0 = rng.normal(0.0, 1.0, n)
    vb = _row_pattern_bounds(rng, x0, rng.random(n))
    cb = _row_bounds(rng, _csr_rowdot(a, x0))
    cost = rng.normal(0.0, 1.0, n)
    return QpProblem(quad=quad, cost=cost, constraint_matrix=a, var_bounds=vb, con_bounds=cb,
                     name=f"banded-n{n}-m{m}-w{half_width}-s{seed}{'-diag' if diagonal_q else ''}")
