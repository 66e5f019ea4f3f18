"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the PDHCG-II solve path.

Restates the reference algorithm (``/root/reference/pkg/src/anchorqp``,
cited below as ``aq/<file>:<line>``) with numpy for the vector algebra and
``oracle/kernels.c`` (a line-for-line-order restatement of the Cython
kernels, built by ``oracle/build_oracle.sh``) for the sparse products, so it
reproduces the reference's trajectory bit for bit: status, outer/inner
counts and objectives equal the reference's golden runs exactly
(``tests/test_oracle.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg use this module, and only as the checker / the CPU baseline; the product
package never imports it.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["bash", os.path.join(HERE, "build_oracle.sh")], check=True)
        L = C.CDLL(LIB)
        P, I, D = C.c_void_p, C.c_int64, C.c_double
        L.orc_csr_matvec.argtypes = [P, P, P, P, I, P]
        L.orc_csr_matvec_t.argtypes = [P, P, P, P, I, I, P]
        L.orc_sym_matvec.argtypes = [P, P, P, P, I, P]
        L.orc_clamp.argtypes = [P, P, P, I, P]
        L.orc_cone_project.argtypes = [P, P, I, P]
        L.orc_diag_prox_step.argtypes = [P, P, P, D, P, P, I, P]
        L.orc_natural_res_sq.argtypes = [P, P, P, P, I]
        L.orc_natural_res_sq.restype = D
        L.orc_dual_step.argtypes = [P, P, D, P, P, I, P]
        L.orc_lincomb3.argtypes = [D, P, D, P, D, P, I, P]
        L.orc_axpby.argtypes = [D, P, D, P, I, P]
        for f in ("orc_csr_matvec", "orc_csr_matvec_t", "orc_sym_matvec", "orc_clamp", "orc_cone_project",
                  "orc_diag_prox_step", "orc_dual_step", "orc_lincomb3", "orc_axpby"):
            getattr(L, f).restype = None
        _lib = L
    return _lib


def _a(x, dt=np.float64):
    return np.ascontiguousarray(x, dtype=dt)


# ---------------------------------------------------------------- kernels (aq/_kernels/_core.pyx)
def csr_matvec(ptr, idx, val, x, rows):                  # _core.pyx:29-42
    ptr, idx, val, x = _a(ptr, np.int64), _a(idx, np.int64), _a(val), _a(x)
    out = np.empty(rows)
    lib().orc_csr_matvec(ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, x.ctypes.data, rows, out.ctypes.data)
    return out


def csr_matvec_t(ptr, idx, val, x, cols):                # _core.pyx:45-59
    ptr, idx, val, x = _a(ptr, np.int64), _a(idx, np.int64), _a(val), _a(x)
    out = np.empty(cols)
    lib().orc_csr_matvec_t(ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, x.ctypes.data, len(ptr) - 1, cols,
                           out.ctypes.data)
    return out


def sym_matvec(ptr, idx, val, x):                        # _core.pyx:62-80
    ptr, idx, val, x = _a(ptr, np.int64), _a(idx, np.int64), _a(val), _a(x)
    out = np.empty(len(x))
    lib().orc_sym_matvec(ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, x.ctypes.data, len(x), out.ctypes.data)
    return out


def clamp(x, lo, hi):                                    # _core.pyx:83-92
    x, lo, hi = _a(x), _a(lo), _a(hi)
    out = np.empty(len(x))
    lib().orc_clamp(x.ctypes.data, lo.ctypes.data, hi.ctypes.data, len(x), out.ctypes.data)
    return out


def cone_project(z, codes):                              # _core.pyx:95-115
    z, codes = _a(z), _a(codes, np.int8)
    out = np.empty(len(z))
    lib().orc_cone_project(z.ctypes.data, codes.ctypes.data, len(z), out.ctypes.data)
    return out


def diag_prox_step(xk, q, lin, tau, lo, hi):             # _core.pyx:118-128
    xk, q, lin, lo, hi = _a(xk), _a(q), _a(lin), _a(lo), _a(hi)
    out = np.empty(len(xk))
    lib().orc_diag_prox_step(xk.ctypes.data, q.ctypes.data, lin.ctypes.data, float(tau), lo.ctypes.data,
                             hi.ctypes.data, len(xk), out.ctypes.data)
    return out


def natural_res_sq(x, g, lo, hi):                        # _core.pyx:131-142
    x, g, lo, hi = _a(x), _a(g), _a(lo), _a(hi)
    return lib().orc_natural_res_sq(x.ctypes.data, g.ctypes.data, lo.ctypes.data, hi.ctypes.data, len(x))


def dual_step(y, ax, sigma, lo, hi):                     # _core.pyx:145-157
    y, ax, lo, hi = _a(y), _a(ax), _a(lo), _a(hi)
    out = np.empty(len(y))
    lib().orc_dual_step(y.ctypes.data, ax.ctypes.data, float(sigma), lo.ctypes.data, hi.ctypes.data, len(y),
                        out.ctypes.data)
    return out


def lincomb3(a, x, b, y, c, z):                          # _core.pyx:160-170
    x, y, z = _a(x), _a(y), _a(z)
    out = np.empty(len(x))
    lib().orc_lincomb3(a, x.ctypes.data, b, y.ctypes.data, c, z.ctypes.data, len(x), out.ctypes.data)
    return out


def axpby(a, x, b, y):                                   # _core.pyx:173-182
    x, y = _a(x), _a(y)
    out = np.empty(len(x))
    lib().orc_axpby(a, x.ctypes.data, b, y.ctypes.data, len(x), out.ctypes.data)
    return out


# ---------------------------------------------------------------- model (aq/model.py)
ZERO, NONNEG, NONPOS, FREE = 0, 1, 2, 3
_TABLES = {  # (lower finite, upper finite) -> code; aq/model.py:85-112
    "dual_y": (ZERO, NONNEG, NONPOS, FREE),
    "dual_r": (ZERO, NONPOS, NONNEG, FREE),
    "recession": (FREE, NONPOS, NONNEG, ZERO),
}


def cones(lo, hi, side):
    key = np.isfinite(lo).astype(np.int64) * 2 + np.isfinite(hi).astype(np.int64)
    return np.asarray(_TABLES[side], dtype=np.int8)[key]


def support(z, lo, hi):                                  # aq/model.py:57-71
    pos, neg = z > 0, z < 0
    if np.any(pos & np.isinf(hi)) or np.any(neg & np.isinf(lo)):
        return float("inf")
    return float(hi[pos] @ z[pos] + lo[neg] @ z[neg])


def linf(v):                                             # aq/certify.py:50-51
    return float(np.abs(v).max()) if len(v) else 0.0


def bound_scale(lo, hi):                                 # aq/certify.py:54-60
    s = 0.0
    for arr in (lo, hi):
        f = arr[np.isfinite(arr)]
        if f.size:
            s = max(s, float(np.abs(f).max()))
    return s


class Instance:
    """Raw arrays of one QpProblem (works on this repo's or the reference's objects)."""

    def __init__(self, p):
        a = p.constraint_matrix
        self.n, self.m = len(p.cost), a.rows
        self.a = (a.indptr, a.indices, a.data)
        self.c = _a(p.cost)
        self.vlo, self.vhi = _a(p.var_bounds.lower), _a(p.var_bounds.upper)
        self.clo, self.chi = _a(p.con_bounds.lower), _a(p.con_bounds.upper)
        q = p.quad
        self.kind = q.kind
        if q.kind == "diagonal":
            self.qd = _a(q.values)
        elif q.kind == "sparse":
            self.qp = (q.upper.indptr, q.upper.indices, q.upper.data, _a(q.diag))
        else:
            self.qp = (q.p.upper.indptr, q.p.upper.indices, q.p.upper.data, _a(q.p.diag))
            self.r = (q.r.indptr, q.r.indices, q.r.data, q.r.rows)
        self.cone_y = cones(self.clo, self.chi, "dual_y")
        self.cone_r = cones(self.vlo, self.vhi, "dual_r")
        self.recc_x = cones(self.vlo, self.vhi, "recession")
        self.recc_s = cones(self.clo, self.chi, "recession")

    # aq/linalg.py:99-105, 164-165, 210-213, 251-254
    def ax(self, x):
        return csr_matvec(*self.a, x, self.m)

    def aty(self, y):
        return csr_matvec_t(*self.a, y, self.n)

    def qx(self, x):
        if self.kind == "diagonal":
            return self.qd * x
        ptr, idx, val, _ = self.qp
        px = sym_matvec(ptr, idx, val, x)
        if self.kind == "sparse":
            return px
        rp, ri, rv, k = self.r
        rx = csr_matvec(rp, ri, rv, x, k)
        return px + csr_matvec_t(rp, ri, rv, rx, self.n)

    def diag_bound(self):                                # aq/linalg.py:167,215,256
        if self.kind == "diagonal":
            return float(self.qd.max(initial=0.0))
        d = self.qp[3]
        if self.kind == "sparse":
            return float(d.max(initial=0.0))
        rp, ri, rv, _ = self.r
        return float((d + np.bincount(ri, weights=rv ** 2, minlength=self.n)).max(initial=0.0))

    def inf_norm_bound(self):                            # aq/linalg.py:170,218-220,260-263
        if self.kind == "diagonal":
            return self.diag_bound()
        ptr, idx, val, d = self.qp
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(ptr))
        acc = (np.bincount(rows, weights=np.abs(val), minlength=self.n)
               + np.bincount(idx, weights=np.abs(val), minlength=self.n) - np.abs(d))
        b = float(acc.max(initial=0.0))
        if self.kind == "sparse":
            return b
        rp, ri, rv, k = self.r
        rrows = np.repeat(np.arange(k, dtype=np.int64), np.diff(rp))
        r_one = float(np.bincount(ri, weights=np.abs(rv), minlength=self.n).max(initial=0.0))
        r_inf = float(np.bincount(rrows, weights=np.abs(rv), minlength=k).max(initial=0.0))
        return b + r_one * r_inf


def estimate_norm(inst, iters=100, seed=0):             # aq/linalg.py:287-312
    if len(inst.a[2]) == 0:
        return None
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(inst.n)
    for _ in range(8):
        nv = np.linalg.norm(v)
        if nv > 0 and np.linalg.norm(inst.ax(v / nv)) > 0:
            break
        v = rng.standard_normal(inst.n)
    else:
        return None
    v /= np.linalg.norm(v)
    for _ in range(iters):
        w = inst.aty(inst.ax(v))
        nw = np.linalg.norm(w)
        if nw == 0.0:
            break
        v = w / nw
    return float(np.linalg.norm(inst.ax(v)))


# ---------------------------------------------------------------- certify (aq/certify.py)
def residuals(inst, x, y):                               # aq/certify.py:63-95
    ax, qx, aty = inst.ax(x), inst.qx(x), inst.aty(y)
    r = qx + inst.c + aty
    pviol = linf(ax - np.minimum(np.maximum(ax, inst.clo), inst.chi))
    r_primal = pviol / (1.0 + bound_scale(inst.clo, inst.chi))
    rp = cone_project(r, inst.cone_r)
    r_dual = linf(r - rp) / (1.0 + max(linf(qx), linf(aty), linf(inst.c)))
    p_r = support(-rp, inst.vlo, inst.vhi)
    p_y = support(cone_project(y, inst.cone_y), inst.clo, inst.chi)
    xqx, cx = float(x @ qx), float(inst.c @ x)
    gap = abs(xqx + cx + p_r + p_y) / (1.0 + max(abs(0.5 * xqx + cx), abs(0.5 * xqx + p_r + p_y)))
    return dict(r_primal=r_primal, r_dual=r_dual, r_gap=gap, primal_objective=0.5 * xqx + cx,
                dual_objective=-p_r - 0.5 * xqx - p_y, dual_slack=r, kkt=max(r_primal, r_dual, gap))


def primal_ray(inst, dy, eps_inf):                       # aq/certify.py:109-133
    ray = cone_project(_a(dy), inst.cone_y)
    nrm = linf(ray)
    if nrm == 0.0 or not math.isfinite(nrm):
        return None
    ray = ray / nrm
    at = inst.aty(ray)
    atp = cone_project(at, inst.cone_r)
    viol = linf(at - atp)
    b = support(-atp, inst.vlo, inst.vhi) + support(ray, inst.clo, inst.chi)
    if not math.isfinite(b) or b >= 0.0:
        return None
    if viol <= eps_inf * -b and viol <= 1e-10 * (1.0 + linf(at)):
        return ("primal_ray", ray, viol, -b)
    return None


def dual_ray(inst, dx, eps_tol, eps_inf, gamma):         # aq/certify.py:136-164
    dx = _a(dx)
    nrm = linf(dx)
    if nrm == 0.0 or not math.isfinite(nrm):
        return None
    d = dx / nrm
    imp = float(inst.c @ d)
    if not imp < -eps_tol:
        return None
    ad = inst.ax(d)
    viol = max(linf(d - cone_project(d, inst.recc_x)), linf(ad - cone_project(ad, inst.recc_s)),
               linf(inst.qx(d)) / gamma)
    if viol <= eps_inf:
        return ("dual_ray", d, viol, imp)
    return None


# ---------------------------------------------------------------- inner (aq/inner.py)
def bb_solve(inst, lin, center, tau, target, max_inner):  # aq/inner.py:84-134
    lo, hi = inst.vlo, inst.vhi

    def grad(x):                                          # aq/inner.py:61-62
        return inst.qx(x) + lin + (x - center) / tau

    def phi_of(x, g):                                     # aq/inner.py:64-66
        return 0.5 * float(x @ g + lin @ x - ((x - center) @ center) / tau)

    x = clamp(center, lo, hi)
    g = grad(x)
    res = math.sqrt(natural_res_sq(x, g, lo, hi))
    phi = phi_of(x, g)
    best = (phi, x, res)
    if res <= target:
        return x, 0
    a0 = tau / (1.0 + tau * inst.diag_bound())
    alpha, t = a0, 0
    for t in range(1, max_inner + 1):
        xn = clamp(x - alpha * g, lo, hi)
        gn = grad(xn)
        res = math.sqrt(natural_res_sq(xn, gn, lo, hi))
        phi = phi_of(xn, gn)
        if phi < best[0]:
            best = (phi, xn, res)
        s, v = xn - x, gn - g
        sv = float(s @ v)
        if sv > 0.0:
            alpha = float(s @ s) / sv if t % 2 == 1 else sv / float(v @ v)
            alpha = min(max(alpha, 1e-10), 1e10)
        else:
            alpha = a0
        x, g = xn, gn
        if res <= target:
            break
    noise = 64.0 * np.finfo(np.float64).eps * (1.0 + abs(best[0]))
    if res <= target and phi <= best[0] + noise:
        return x, t
    if phi <= best[0]:
        return x, t
    return best[1], t


# ---------------------------------------------------------------- engine (aq/engine.py)
def solve(problem, params, max_seconds=None):
    """aq/engine.py:339-498.  ``params`` is any object with the SolverParams
    fields.  Returns a dict (status, x, y, report, outer, inner, restarts,
    seconds, certificate).  ``max_seconds`` (oracle-only) stops a bounded
    sample early and reports status "sample"."""
    t0 = time.monotonic()
    inst = problem if isinstance(problem, Instance) else Instance(problem)
    P, R, IN = params, params.restart, params.inner
    x = clamp(np.zeros(inst.n), inst.vlo, inst.vhi)      # aq/engine.py:176-177
    y = np.zeros(inst.m)
    nrm = estimate_norm(inst, P.norm_iters, P.norm_seed)
    eta = 1e8 if nrm is None else P.eta_scale / nrm     # aq/engine.py:178-183
    st = dict(x=x, y=y, xp=x.copy(), yp=y.copy(), ax=x.copy(), ay=y.copy(), k=0, rnd=0, omega=P.omega0,
              theta=P.theta, integ=0.0, eprev=0.0, tol=IN.initial if IN.adaptive else IN.fixed_tol,
              brs=math.inf, lck=math.inf)
    gamma = P.gamma_sys if P.gamma_sys is not None else 1.0 + inst.inf_norm_bound()
    n_out = n_in = restarts = 0

    def out(status, rep, cert, xe):
        return dict(status=status, x=xe, y=st["y"], report=rep, certificate=cert, outer=n_out, inner=n_in,
                    restarts=restarts, seconds=time.monotonic() - t0)

    def anchor_here(kkt):                                 # aq/engine.py:291-300, 322-333
        st["ax"], st["ay"] = st["x"].copy(), st["y"].copy()
        st["xp"], st["yp"] = st["x"].copy(), st["y"].copy()
        st["k"] = 0
        st["rnd"] += 1
        st["brs"] = st["lck"] = kkt

    def rollback():                                       # aq/engine.py:303-319
        st["x"], st["y"] = st["ax"].copy(), st["ay"].copy()
        st["xp"], st["yp"] = st["ax"].copy(), st["ay"].copy()
        st["k"] = 0
        st["rnd"] += 1
        st["theta"] = st["theta"] / 2.0 if st["theta"] >= 1e-2 else 0.0
        st["lck"] = st["brs"]

    def pid():                                            # aq/engine.py:260-281
        dx = float(np.linalg.norm(st["x"] - st["ax"]))
        dy = float(np.linalg.norm(st["y"] - st["ay"]))
        if dx <= 0.0 or dy <= 0.0 or not (math.isfinite(dx) and math.isfinite(dy)):
            return st["omega"]
        e = math.log(st["omega"] * dx / dy)
        if not math.isfinite(e):
            return st["omega"]
        kp, ki, kd = P.pid_gains
        integ = min(max(st["integ"] + e, -10.0), 10.0)
        lw = math.log(st["omega"]) - (kp * e + ki * integ + kd * (e - st["eprev"]))
        st["integ"], st["eprev"] = integ, e
        return min(max(math.exp(lw), 1e-6), 1e6)

    xe = clamp(st["x"], inst.vlo, inst.vhi)
    rep = residuals(inst, xe, st["y"])
    st["brs"] = st["lck"] = rep["kkt"]
    if rep["kkt"] <= P.eps_tol:
        return out("optimal", rep, None, xe)
    xl, yl = st["x"].copy(), st["y"].copy()
    best_seen, stall, probe_until = rep["kkt"], 0, 0
    xb, yb, blen, xap, yap = np.zeros(inst.n), np.zeros(inst.m), 0, None, None
    while n_out < P.iter_limit:
        probing = n_out < probe_until
        tau, sigma = eta / st["omega"], eta * st["omega"]
        lin = inst.c + inst.aty(st["y"])                  # aq/engine.py:214
        if inst.kind == "diagonal":
            xplus, t = diag_prox_step(st["x"], inst.qd, lin, tau, inst.vlo, inst.vhi), 0
        else:
            target = min(st["tol"], 1e-12) if probing else st["tol"]
            xplus, t = bb_solve(inst, lin, st["x"], tau, target, IN.max_inner)
        xbar = axpby(2.0, xplus, -1.0, st["x"])           # aq/engine.py:222-226
        yplus = dual_step(st["y"], inst.ax(xbar), sigma, inst.clo, inst.chi)
        if probing or not P.halpern:                      # aq/engine.py:230-245, 400-403
            zx, zy = xplus, yplus
        else:
            k, th = st["k"], st["theta"]
            ca, cb = (1.0 + th) * ((k + 1.0) / (k + 2.0)), (1.0 + th) * (1.0 / (k + 2.0))
            zx = lincomb3(ca, xplus, cb, st["ax"], -th, st["xp"])
            zy = lincomb3(ca, yplus, cb, st["ay"], -th, st["yp"])
        move = float(np.linalg.norm(zx - st["x"]))
        n_out += 1
        n_in += t
        if not math.isfinite(move):                       # aq/engine.py:407-417
            rollback()
            xl, yl, probe_until, xap, yap = st["x"].copy(), st["y"].copy(), 0, None, None
            xb[:] = 0.0
            yb[:] = 0.0
            blen = 0
            continue
        if IN.adaptive:                                   # aq/inner.py:41-48
            st["tol"] = min(st["tol"], max(IN.scale * st["omega"] * move / tau, IN.floor))
        st["xp"], st["yp"], st["x"], st["y"] = st["x"], st["y"], zx, zy
        if not probing:
            st["k"] += 1
        xb += zx
        yb += zy
        blen += 1
        at_cap = (not probing) and R.enabled and st["k"] >= R.max_round_len
        if not (n_out % P.check_every == 0 or at_cap or n_out == P.iter_limit):
            continue
        xe = clamp(st["x"], inst.vlo, inst.vhi)          # aq/engine.py:436-494
        rep = residuals(inst, xe, st["y"])
        kkt = rep["kkt"]
        if kkt <= P.eps_tol:
            return out("optimal", rep, None, xe)
        xa, ya = xb / blen, yb / blen
        xb, yb, blen = np.zeros(inst.n), np.zeros(inst.m), 0
        dys, dxs = [st["y"] - yl], [st["x"] - xl]
        if yap is not None:
            dys.insert(0, ya - yap)
            dxs.insert(0, xa - xap)
        xap, yap = xa, ya
        for d in dys:
            cert = primal_ray(inst, d, P.eps_inf)
            if cert:
                return out("primal_infeasible", rep, cert, xe)
        for d in dxs:
            cert = dual_ray(inst, d, P.eps_tol, P.eps_inf, gamma)
            if cert:
                return out("dual_infeasible", rep, cert, xe)
        xl, yl = st["x"].copy(), st["y"].copy()
        if math.isfinite(kkt) and kkt < 0.99 * best_seen:
            best_seen, stall = min(best_seen, kkt), 0
        else:
            stall += 1
        if probing:
            if n_out >= probe_until:
                if stall == 0:
                    anchor_here(kkt)
                else:
                    probe_until = n_out + R.max_round_len
        elif stall >= 8:
            probe_until = n_out + R.max_round_len
        elif not math.isfinite(kkt) or kkt > 100.0 * st["brs"]:
            rollback()
            xl, yl = st["x"].copy(), st["y"].copy()
        elif R.enabled and (st["k"] >= R.max_round_len or kkt <= R.beta_sufficient * st["brs"]
                            or (kkt <= R.beta_necessary * st["brs"] and kkt > st["lck"])):
            if kkt < st["brs"]:
                st["omega"] = pid()
            anchor_here(kkt)
            restarts += 1
        else:
            st["lck"] = kkt
        if P.time_limit is not None and time.monotonic() - t0 >= P.time_limit:
            return out("time_limit", rep, None, xe)
        if max_seconds is not None and time.monotonic() - t0 >= max_seconds:
            return out("sample", rep, None, xe)
    xe = clamp(st["x"], inst.vlo, inst.vhi)
    return out("iteration_limit", residuals(inst, xe, st["y"]), None, xe)
