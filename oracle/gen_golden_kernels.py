"""TEST INFRASTRUCTURE ONLY: record the reference's own kernel outputs
(Cython backend of the built reference in oracle/_ref) on seeded inputs, plus
the hashes of the generator instances, as committed fixtures under
tests/golden/.  Re-run with:  python oracle/gen_golden_kernels.py
"""
import hashlib
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
import instances  # noqa: E402
import refbridge  # noqa: E402

aq = refbridge.load_reference()
from anchorqp._kernels import _core  # noqa: E402

rng = np.random.default_rng(20261017)
out = {}


def csr(rows, cols, dens):
    m = sp.random(rows, cols, density=dens, random_state=rng, data_rvs=lambda k: rng.uniform(-1, 1, k)).tocsr()
    m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data


for t, (r, c, d) in enumerate([(1, 1, 1.0), (9, 14, 0.4), (200, 150, 0.05), (3, 5000, 0.5), (1500, 1200, 0.01)]):
    ip, ix, dv = csr(r, c, d)
    x, y = rng.standard_normal(c), rng.standard_normal(r)
    y[rng.random(r) < 0.2] = 0.0  # exercise the skip-zero-row branch of _core.pyx:56
    out[f"mv{t}_indptr"], out[f"mv{t}_indices"], out[f"mv{t}_data"] = ip, ix, dv
    out[f"mv{t}_x"], out[f"mv{t}_y"] = x, y
    out[f"mv{t}_ax"] = _core.csr_matvec(ip, ix, dv, x, r)
    out[f"mv{t}_aty"] = _core.csr_matvec_t(ip, ix, dv, y, c)
for t, n in enumerate([1, 7, 120, 900]):
    b = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.1)
    full = b + b.T + np.diag(rng.uniform(0, 1, n))
    u = sp.triu(sp.csr_matrix(full)).tocsr()
    u.sort_indices()
    x = rng.standard_normal(n)
    out[f"sym{t}_indptr"], out[f"sym{t}_indices"], out[f"sym{t}_data"] = u.indptr.astype(np.int64), u.indices.astype(np.int64), u.data
    out[f"sym{t}_diag"], out[f"sym{t}_x"] = np.diag(full).copy(), x
    out[f"sym{t}_out"] = _core.sym_matvec(out[f"sym{t}_indptr"], out[f"sym{t}_indices"], u.data, out[f"sym{t}_diag"], x)
n = 777
x, g, q, lin = rng.standard_normal(n), rng.standard_normal(n), rng.uniform(0, 2, n), rng.standard_normal(n)
lo = np.where(rng.random(n) < 0.3, -np.inf, -0.6)
hi = np.where(rng.random(n) < 0.3, np.inf, 0.7)
codes = rng.integers(0, 4, n).astype(np.int8)
out.update(v_x=x, v_g=g, v_q=q, v_lin=lin, v_lo=lo, v_hi=hi, v_codes=codes)
out["k_clamp"] = _core.clamp(x, lo, hi)
out["k_cone"] = _core.cone_project(x, codes)
out["k_prox"] = _core.diag_prox_step(x, q, lin, 0.37, lo, hi)
out["k_natres"] = np.array([_core.natural_res_sq(x, g, lo, hi)])
out["k_dual"] = _core.dual_step(x, g, 1.7, lo, hi)
out["k_lin3"] = _core.lincomb3(0.3, x, 0.6, g, -0.25, lin)
out["k_axpby"] = _core.axpby(2.0, x, -1.0, g)
out["k_support"] = np.array([aq.support_p(x * (np.isfinite(lo) & np.isfinite(hi)), aq.Bounds(lo, hi))])
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "kernels.npz"), **out)


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


hashes = {}
for args in [(2000, 1000, "sparse", 0.01, 0), (40, 20, "diagonal", 0.3, 1), (30, 15, "low_rank", 0.3, 4),
             (300, 150, "sparse", 0.05, 7)]:
    hashes["random_qp" + repr(args)] = digest(aq.random_qp(*args))
a, b = aq.random_lasso_data(30, 20, density=0.3, seed=2)
hashes["make_lasso_qp(random_lasso_data(30,20,0.3,2))"] = digest(aq.make_lasso_qp(a, b))
with open(os.path.join(ROOT, "tests", "golden", "generator_hashes.json"), "w") as f:
    json.dump(hashes, f, indent=1)
print("wrote kernels.npz and generator_hashes.json")
