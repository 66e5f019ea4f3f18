import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2602_23967_b200 as ours
from paper_2602_23967_b200 import _native as nat, certify
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem, DeviceSolver
for args in [(40, 20, "diagonal", 0.3, 1)]:
    p = ours.random_qp(*args)
    dev = DeviceProblem(p, DeviceContext.get())
    sol = DeviceSolver(dev, eps_tol=1e-8, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9, diag_bound=1.0, adaptive=True, max_inner=200, halpern=True)
    sc = nat.Scalars(); sc.eta = 0.5; sc.omega = 1.0; sc.inner_tol = 1e-2
    sol.init(sc)
    cr = sol.check(False)
    x = np.clip(np.zeros(p.n), p.var_bounds.lower, p.var_bounds.upper)
    A = p.constraint_matrix.to_scipy()
    lo, hi = p.con_bounds.lower, p.con_bounds.upper
    for name, xx in [("xeval", x), ("zero", np.zeros(p.n))]:
        ax = A @ xx
        viol = np.abs(ax - np.minimum(np.maximum(ax, lo), hi))
        print(name, "viol sorted", np.sort(viol)[::-1][:6])
    for name, (l2, h2) in [("var-bounds-prefix", (p.var_bounds.lower[:p.m], p.var_bounds.upper[:p.m]))]:
        ax = A @ x
        viol = np.abs(ax - np.minimum(np.maximum(ax, l2), h2))
        print(name, np.sort(viol)[::-1][:4])
    print("dev viol", cr.primal_viol, "qx_inf", cr.qx_inf, "aty", cr.aty_inf, "py", cr.py_pos, cr.py_neg, cr.py_bad)
    axd = sol.read(8); ax = A @ x
    print("ax equal", np.array_equal(axd, ax), np.abs(axd-ax).max())
    viol = np.abs(ax - np.minimum(np.maximum(ax, lo), hi))
    print("viol by row", np.round(viol, 3))
    print("clo eq", np.array_equal(sol.read(9), lo), "chi eq", np.array_equal(sol.read(10), hi))
    print("dev per-row viol", np.round(sol.read(11), 3))
    import paper_2602_23967_b200._native as N, ctypes as C
    out = np.empty(p.n); 
    print("acc after row", np.round(sol.read(12)[:p.m], 3))
    print("thread of row", sol.read(13)[:p.m])
    print("con lo", lo[:6], "hi", hi[:6])
