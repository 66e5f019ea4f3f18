"""The "cuda" kernel backend: ctypes stub over libaqp's registry entry points.

Same ten names and signatures as the reference registry
(``anchorqp/_kernels/__init__.py:16-27`` / ``_core.pyx:29-182``): numpy in,
fresh numpy out, inputs borrowed read-only.  Each call runs on the B200
(host->HBM copy, sm_100a kernel, HBM->host copy).  Registering this module
into the reference's ``_BACKENDS`` makes its own kernel tests run on the GPU
(see INTEGRATION.md); this package's containers call it directly.

The CSR products use libaqp's strict plan (one thread per row, sequential
column order), so ``csr_matvec`` / ``csr_matvec_t`` / ``sym_matvec`` equal the
Cython kernels bit for bit.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat

ZERO, NONNEG, NONPOS, FREE = 0, 1, 2, 3


def _lib():
    return nat.load()


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def csr_matvec(indptr, indices, data, x, nrows):
    indptr, indices, data, x = _i64(indptr), _i64(indices), _f64(data), _f64(x)
    out = np.empty(int(nrows), dtype=np.float64)
    nat.check(_lib().aqp_csr_matvec(indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, x.ctypes.data,
                                    int(nrows), len(x), out.ctypes.data), "csr_matvec")
    return out


def csr_matvec_t(indptr, indices, data, x, ncols):
    indptr, indices, data, x = _i64(indptr), _i64(indices), _f64(data), _f64(x)
    out = np.empty(int(ncols), dtype=np.float64)
    nat.check(_lib().aqp_csr_matvec_t(indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, x.ctypes.data,
                                      len(indptr) - 1, int(ncols), out.ctypes.data), "csr_matvec_t")
    return out


def sym_matvec(indptr, indices, data, diag, x):
    indptr, indices, data, diag, x = _i64(indptr), _i64(indices), _f64(data), _f64(diag), _f64(x)
    out = np.empty(len(x), dtype=np.float64)
    nat.check(_lib().aqp_sym_matvec(indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, diag.ctypes.data,
                                    x.ctypes.data, len(x), out.ctypes.data), "sym_matvec")
    return out


def clamp(x, lo, hi):
    x, lo, hi = _f64(x), _f64(lo), _f64(hi)
    out = np.empty(len(x), dtype=np.float64)
    nat.check(_lib().aqp_clamp(x.ctypes.data, lo.ctypes.data, hi.ctypes.data, len(x), out.ctypes.data), "clamp")
    return out


def cone_project(z, codes):
    z = _f64(z)
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    out = np.empty(len(z), dtype=np.float64)
    nat.check(_lib().aqp_cone_project(z.ctypes.data, codes.ctypes.data, len(z), out.ctypes.data), "cone_project")
    return out


def diag_prox_step(xk, q, linear, tau, lo, hi):
    xk, q, linear, lo, hi = _f64(xk), _f64(q), _f64(linear), _f64(lo), _f64(hi)
    out = np.empty(len(xk), dtype=np.float64)
    nat.check(_lib().aqp_diag_prox_step(xk.ctypes.data, q.ctypes.data, linear.ctypes.data, float(tau),
                                        lo.ctypes.data, hi.ctypes.data, len(xk), out.ctypes.data), "diag_prox_step")
    return out


def natural_res_sq(x, g, lo, hi):
    x, g, lo, hi = _f64(x), _f64(g), _f64(lo), _f64(hi)
    out = np.empty(1, dtype=np.float64)
    nat.check(_lib().aqp_natural_res_sq(x.ctypes.data, g.ctypes.data, lo.ctypes.data, hi.ctypes.data, len(x),
                                        out.ctypes.data), "natural_res_sq")
    return float(out[0])


def dual_step(y, ax, sigma, lo, hi):
    y, ax, lo, hi = _f64(y), _f64(ax), _f64(lo), _f64(hi)
    out = np.empty(len(y), dtype=np.float64)
    nat.check(_lib().aqp_dual_step(y.ctypes.data, ax.ctypes.data, float(sigma), lo.ctypes.data, hi.ctypes.data,
                                   len(y), out.ctypes.data), "dual_step")
    return out


def lincomb3(a, x, b, y, c, z):
    x, y, z = _f64(x), _f64(y), _f64(z)
    out = np.empty(len(x), dtype=np.float64)
    nat.check(_lib().aqp_lincomb3(float(a), x.ctypes.data, float(b), y.ctypes.data, float(c), z.ctypes.data,
                                  len(x), out.ctypes.data), "lincomb3")
    return out


def axpby(a, x, b, y):
    x, y = _f64(x), _f64(y)
    out = np.empty(len(x), dtype=np.float64)
    nat.check(_lib().aqp_axpby(float(a), x.ctypes.data, float(b), y.ctypes.data, len(x), out.ctypes.data), "axpby")
    return out


# ---- helpers used by the host containers (not registry names) -------------
def support_p(z, lo, hi) -> float:
    z, lo, hi = _f64(z), _f64(lo), _f64(hi)
    out = np.empty(1, dtype=np.float64)
    nat.check(_lib().aqp_support_p(z.ctypes.data, lo.ctypes.data, hi.ctypes.data, len(z), out.ctypes.data),
              "support_p")
    return float(out[0])


def quad_apply(q, x):
    """Q @ x for the three operator variants (linalg.py:164,210,251) on the device."""
    if q.kind == "diagonal":
        return _diag_apply(q.values, x)
    if q.kind == "sparse":
        u = q.upper
        return sym_matvec(u.indptr, u.indices, u.data, q.diag, x)
    rx = csr_matvec(q.r.indptr, q.r.indices, q.r.data, x, q.r.rows)
    px = quad_apply(q.p, x)
    rt = csr_matvec_t(q.r.indptr, q.r.indices, q.r.data, rx, q.r.cols)
    return axpby(1.0, px, 1.0, rt)


def _diag_apply(values, x):
    # q * x as the CSR product of diag(values): one product per row, added to
    # 0.0 -- the value numpy's `values * x` gives
    n = len(values)
    return csr_matvec(np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), values, x, n)


def estimate_norm(a, iters: int, seed: int) -> float:
    """Power-iteration norm estimate of ``a`` on the device (linalg.py:287-312)."""
    from .device import DeviceContext, DeviceProblem, DeviceSolver
    from .errors import ZeroMatrix
    from .linalg import DiagonalQuad
    from .model import Bounds, QpProblem

    prob = QpProblem(quad=DiagonalQuad(np.zeros(a.cols)), cost=np.zeros(a.cols), constraint_matrix=a,
                     var_bounds=Bounds.free(a.cols), con_bounds=Bounds.free(a.rows))
    dev = DeviceProblem(prob, DeviceContext.get())
    sol = DeviceSolver(dev, eps_tol=1e-6, eps_inf=1e-9, gamma_sys=1.0, tol_scale=5e-4, tol_floor=1e-9,
                       diag_bound=0.0, adaptive=True, max_inner=200, halpern=True)
    rng = np.random.default_rng(seed)
    for _ in range(8):
        est, annihilated = sol.estimate_norm(rng.standard_normal(a.cols), iters)
        if not annihilated:
            return est
    raise ZeroMatrix("power iteration start vector annihilated by A")
