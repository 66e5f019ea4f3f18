"""Ad-hoc GPU shakedown: registry kernels vs the Cython reference, then solves."""
import os, sys, time, json, traceback
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import scipy.sparse as sp
import refbridge, instances
aq = refbridge.load_reference()
import paper_2602_23967_b200 as ours
from paper_2602_23967_b200 import kernels as K
from anchorqp._kernels import _core

rng = np.random.default_rng(0)
def rcsr(r, c, d=0.3):
    m = sp.random(r, c, density=d, random_state=rng).tocsr(); m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data
ok = True
for (r, c) in [(1, 1), (7, 13), (100, 80), (3000, 2000), (5, 20000)]:
    ip, ix, dv = rcsr(r, c, 0.3 if r * c < 1e6 else 0.2)
    x = rng.standard_normal(c); y = rng.standard_normal(r)
    a = K.csr_matvec(ip, ix, dv, x, r); b = _core.csr_matvec(ip, ix, dv, x, r)
    at = K.csr_matvec_t(ip, ix, dv, y, c); bt = _core.csr_matvec_t(ip, ix, dv, y, c)
    print("matvec", r, c, "bitwise", np.array_equal(a, b), np.array_equal(at, bt), np.abs(a-b).max() if r else 0)
    ok &= np.array_equal(a, b) and np.array_equal(at, bt)
for n in [1, 5, 50, 600, 3000]:
    base = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.2); full = base + base.T
    up = sp.triu(sp.csr_matrix(full)).tocsr(); up.sort_indices()
    x = rng.standard_normal(n)
    a = K.sym_matvec(up.indptr.astype(np.int64), up.indices.astype(np.int64), up.data, np.diag(full).copy(), x)
    b = _core.sym_matvec(up.indptr.astype(np.int64), up.indices.astype(np.int64), up.data, np.diag(full).copy(), x)
    print("sym", n, "bitwise", np.array_equal(a, b), np.abs(a - b).max())
n = 1000
x, g, lo, hi = rng.standard_normal(n), rng.standard_normal(n), np.full(n, -0.5), np.full(n, 0.5)
print("natres", K.natural_res_sq(x, g, lo, hi), _core.natural_res_sq(x, g, lo, hi))
print("clamp eq", np.array_equal(K.clamp(x, lo, hi), _core.clamp(x, lo, hi)))
print("dual_step eq", np.array_equal(K.dual_step(x, g, 1.3, lo, hi), _core.dual_step(x, g, 1.3, lo, hi)))
print("lincomb3 eq", np.array_equal(K.lincomb3(0.3, x, 0.5, g, -0.2, lo), _core.lincomb3(0.3, x, 0.5, g, -0.2, lo)))

def cmp(spec_or_prob, eps=1e-8, label=None, **kw):
    p = instances.build(spec_or_prob) if isinstance(spec_or_prob, str) else spec_or_prob
    rp = refbridge.to_reference(p, aq)
    t = time.time(); r1 = ours.solve(p, ours.SolverParams(eps_tol=eps, **kw)); t1 = time.time() - t
    t = time.time(); r0 = aq.solve(rp, aq.SolverParams(eps_tol=eps, **kw)); t0 = time.time() - t
    print(json.dumps(dict(case=label or str(spec_or_prob), ours=[r1.status.value, r1.outer_iterations, r1.inner_iterations, r1.restarts, r1.report.primal_objective, r1.report.kkt_max, round(t1, 3)],
                          ref=[r0.status.value, r0.outer_iterations, r0.inner_iterations, r0.restarts, r0.report.primal_objective, r0.report.kkt_max, round(t0, 3)])), flush=True)
    return r1, r0

for args in [(8, 5, "sparse", 0.3, 3), (10, 6, "sparse", 0.3, 11), (6, 4, "diagonal", 0.3, 5), (30, 15, "low_rank", 0.3, 4), (40, 20, "diagonal", 0.3, 1)]:
    try:
        cmp(ours.random_qp(*args), label=str(args))
    except Exception:
        traceback.print_exc()
for spec in ["c1:0", "c2:1e4:5e3:0", "c4u:1e3:1", "c4i:1e3:1"]:
    try:
        cmp(spec)
    except Exception:
        traceback.print_exc()
# timing of our C1 solve (warm)
p = instances.build("c1:0")
for _ in range(2):
    t = time.time(); r = ours.solve(p, ours.SolverParams(eps_tol=1e-8)); print("C1 ours", r.status.value, r.outer_iterations, r.inner_iterations, time.time() - t)
p = instances.build("c2:1e6:5e5:0")
t = time.time(); r = ours.solve(p, ours.SolverParams(eps_tol=1e-8, iter_limit=256)); print("C2 256 iters", r.status.value, r.outer_iterations, r.inner_iterations, r.report.kkt_max, time.time() - t)
