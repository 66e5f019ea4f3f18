"""Search a C4 base instance whose infeasibility certifies quickly at n=1e5."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, scipy.sparse as sp
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators as g
from paper_2602_23967_b200.linalg import DiagonalQuad, SparseMatrix
from paper_2602_23967_b200.model import Bounds, QpProblem

def pair_from(base, seed):
    a = base.constraint_matrix
    q = base.quad.values.copy(); q[0] = 0.0
    c = base.cost.copy(); c[0] = -1.0
    lo = base.var_bounds.lower.copy(); hi = base.var_bounds.upper.copy(); lo[0], hi[0] = 0.0, np.inf
    a_sp = a.to_scipy().tocsc(); a_sp[:, 0] = 0.0; a0 = a_sp.tocsr(); a0.eliminate_zeros()
    unb = QpProblem(DiagonalQuad(q), c, SparseMatrix.from_scipy(a0), Bounds(lo, hi), base.con_bounds)
    rng = np.random.default_rng(seed + 7919); n = base.n
    cols = np.sort(rng.choice(n, 10, replace=False)); vals = rng.uniform(-1, 1, 10)
    extra = sp.csr_matrix((np.concatenate([vals, vals]), (np.repeat([0, 1], 10), np.concatenate([cols, cols]))), shape=(2, n))
    a1 = sp.vstack([a.to_scipy(), extra], format="csr")
    inf = QpProblem(base.quad, base.cost, SparseMatrix.from_scipy(a1), base.var_bounds,
                    Bounds(np.concatenate([base.con_bounds.lower, [1.0, 2.0]]), np.concatenate([base.con_bounds.upper, [1.0, 2.0]])))
    return unb, inf

def diag_lasso(n, m, seed, per_row=8):
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, (m, per_row)); vals = rng.uniform(-1, 1, (m, per_row))
    a = g._csr_from_rows(m, n, cols, vals)
    x0 = rng.normal(0, 1, n)
    vb = g._row_pattern_bounds(rng, x0, rng.random(n)); cb = g._row_bounds(rng, g._csr_rowdot(a, x0))
    return QpProblem(DiagonalQuad(rng.uniform(0.5, 2.0, n)), rng.normal(0, 1, n), a, vb, cb)

cands = {
  "rqp_diag_m/2": lambda n, s: g.random_qp(n, n // 2, "diagonal", density=10 / n, seed=s),
  "rqp_diag_m/10": lambda n, s: g.random_qp(n, n // 10, "diagonal", density=10 / n, seed=s),
  "banded_diag": lambda n, s: g.banded_qp(n, n // 2, half_width=50, seed=s, diagonal_q=True),
  "diag_lasso_m/2": lambda n, s: diag_lasso(n, n // 2, s),
  "diag_lasso_m/10": lambda n, s: diag_lasso(n, n // 10, s),
}
for name, mk in cands.items():
    for n in (10_000, 100_000):
        base = mk(n, 1)
        for lab, p in zip(("unb", "inf"), pair_from(base, 1)):
            t = time.time()
            r = aq.solve(p, aq.SolverParams(eps_tol=1e-8, iter_limit=300_000))
            print(f"{name:16s} n={n:6d} {lab} {r.status.value:18s} outer={r.outer_iterations:7d} {time.time()-t:6.1f}s", flush=True)
