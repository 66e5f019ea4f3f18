"""Device-side objects: PyTorch owns the HBM, libaqp owns the layout and math.

* :class:`DeviceContext` binds libaqp to a CUDA device and a torch stream.
* :class:`DeviceProblem` uploads a :class:`~.model.QpProblem` (reference
  layouts: int64 CSR + float64) and lets libaqp build the device form -- int32
  CSR of A, an explicit A' and the full symmetric Q, their SpMV work plans
  and the cone codes -- inside one torch-allocated workspace.
* :class:`DeviceSolver` is the iteration state of one ``solve`` call.

Nothing here computes on the host; a missing library or device raises.
"""

from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import _native as nat
from .errors import DeviceError
from .model import QpProblem

_contexts = {}


def _torch():
    try:
        import torch
    except ImportError as exc:  # pragma: no cover - torch is part of the image
        raise DeviceError("PyTorch is required for device buffers") from exc
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device available: the solver has no host fallback")
    return torch


class DeviceContext:
    """libaqp context on (device, current torch stream)."""

    def __init__(self, device: int = 0):
        torch = _torch()
        self.lib = nat.load()
        self.device = int(device)
        torch.cuda.set_device(self.device)
        self.torch = torch
        self.stream = torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        nat.check(self.lib.aqp_ctx_create(self.device, C.c_void_p(self.stream.cuda_stream), C.byref(h)),
                  "aqp_ctx_create")
        self.handle = h

    @classmethod
    def get(cls, device: int = 0) -> "DeviceContext":
        torch = _torch()
        key = (int(device), torch.cuda.current_stream(int(device)).cuda_stream)
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = _contexts[key] = cls(device)
        return ctx

    def empty(self, nbytes: int):
        return self.torch.empty(max(int(nbytes), 1), dtype=self.torch.uint8, device=f"cuda:{self.device}")

    def upload(self, arr: np.ndarray):
        """Device copy of a host array: the library's staged multi-threaded
        pinned pipeline (aqp_h2d, ~45 GB/s) instead of a pageable copy."""
        arr = np.ascontiguousarray(arr)
        t = self.empty(arr.nbytes)
        nat.check(self.lib.aqp_h2d(self.handle, C.c_void_p(t.data_ptr()), C.c_void_p(arr.ctypes.data), arr.nbytes),
                  "aqp_h2d")
        return t


def _full_rows(r) -> bool:
    """Every row of the CSR holds all columns in order (a dense factor)."""
    n = r.cols
    if r.rows == 0 or n == 0 or r.nnz != r.rows * n:
        return False
    if not np.array_equal(np.asarray(r.indptr), np.arange(r.rows + 1, dtype=np.int64) * n):
        return False
    idx = np.asarray(r.indices).reshape(r.rows, n)
    return bool((idx == np.arange(n, dtype=idx.dtype)).all())


class DeviceProblem:
    """HBM copy of one QpProblem (reference model.py:124-165), or -- with
    ``part`` (shard.LocalPart) -- of one rank's row shard of it: only that
    rank's rows of A, A' and Q and its entries of the vectors are uploaded
    and stored (aqp_shard_desc)."""

    def __init__(self, problem: QpProblem, ctx: DeviceContext = None, part=None):
        self.ctx = ctx or DeviceContext.get()
        lib = self.ctx.lib
        p = problem
        a = p.constraint_matrix
        q = p.quad
        keep = []  # upload tensors, alive until create() returns

        def up(arr):
            t = self.ctx.upload(arr)
            keep.append(t)
            return t.data_ptr()

        d = nat.ProblemDesc()
        d.n, d.m = p.n, p.m
        sh = None
        if part is None:
            a_ptr, a_idx, a_val = a.indptr, a.indices, a.data
        else:
            a_ptr, a_idx, a_val = part.a_indptr, part.a_indices, part.a_data
        d.a_indptr, d.a_indices, d.a_data, d.a_nnz = up(a_ptr), up(a_idx), up(a_val), len(a_val)
        host_q = host_r = None
        if q.kind == "diagonal":
            d.quad_kind = nat.QUAD_DIAGONAL
            d.q_values = up(q.values if part is None else part.q_vec)
        else:
            pq = q if q.kind == "sparse" else q.p
            d.quad_kind = nat.QUAD_SPARSE if q.kind == "sparse" else nat.QUAD_SPARSE_LOW_RANK
            if part is None:
                q_ptr, q_idx, q_val, q_diag = pq.upper.indptr, pq.upper.indices, pq.upper.data, pq.diag
            else:
                q_ptr, q_idx, q_val, q_diag = part.q_indptr, part.q_indices, part.q_data, part.q_vec
            d.q_indptr, d.q_indices, d.q_data = up(q_ptr), up(q_idx), up(q_val)
            d.q_nnz = len(q_val)
            d.q_diag = up(q_diag)
            host_q = np.ascontiguousarray(q_ptr, dtype=np.int64)
            if q.kind == "sparse_low_rank":
                r = q.r
                d.r_rows = r.rows
                if part is None:
                    d.r_dense = int(_full_rows(r))
                    r_ptr, r_idx, r_val = r.indptr, r.indices, r.data
                else:
                    d.r_dense = int(part.r_dense)
                    r_ptr, r_idx, r_val = part.r_indptr, part.r_indices, part.r_data
                d.r_indptr = up(r_ptr)
                d.r_indices = 0 if d.r_dense else up(r_idx)  # dense: the indices are implied
                d.r_data, d.r_nnz = up(r_val), len(r_val)
                host_r = np.ascontiguousarray(r_ptr, dtype=np.int64)
        src = p if part is None else None
        d.cost = up(p.cost if src else part.cost)
        d.var_lo = up(p.var_bounds.lower if src else part.var_lo)
        d.var_hi = up(p.var_bounds.upper if src else part.var_hi)
        d.con_lo = up(p.con_bounds.lower if src else part.con_lo)
        d.con_hi = up(p.con_bounds.upper if src else part.con_hi)
        if part is not None:
            me = part.me
            sh = nat.ShardDesc(rank=me.rank, nranks=me.nranks, n0=me.n0, n1=me.n1, m0=me.m0, m1=me.m1,
                               a_row0=me.ywin[0], a_rows=me.ywin[1] - me.ywin[0], q_row0=me.q_row0,
                               a_local_nnz=me.a_local_nnz, at_local_nnz=me.at_local_nnz,
                               q_local_nnz=me.q_local_nnz,
                               nl_cap=max(pl.n1 - pl.n0 for pl in part.plans),
                               ml_cap=max(pl.m1 - pl.m0 for pl in part.plans))
            for k, pl in enumerate(part.plans):
                sh.xw[2 * k], sh.xw[2 * k + 1] = pl.xwin
                sh.yw[2 * k], sh.yw[2 * k + 1] = pl.ywin
            d.shard = C.addressof(sh)
        host_a = np.ascontiguousarray(a_ptr, dtype=np.int64)
        self.timing = {}
        phases = os.environ.get("AQP_PHASES", "") == "1"
        if phases:
            self.ctx.torch.cuda.synchronize()
            t_up = time.perf_counter()
        pb, sb = C.c_size_t(), C.c_size_t()
        nat.check(lib.aqp_problem_sizes(C.byref(d), C.byref(pb), C.byref(sb)), "aqp_problem_sizes")
        self.workspace = self.ctx.empty(pb.value)
        scratch = self.ctx.empty(sb.value)
        h = C.c_void_p()
        rc = lib.aqp_problem_create(
            self.ctx.handle, C.byref(d), host_a.ctypes.data,
            None if host_q is None else host_q.ctypes.data,
            None if host_r is None else host_r.ctypes.data,
            C.c_void_p(self.workspace.data_ptr()), pb.value, C.c_void_p(scratch.data_ptr()), sb.value, C.byref(h))
        nat.check(rc, "aqp_problem_create")
        del scratch, keep
        # SELL-32 copies of the uniform matrices, in memory the upload buffers
        # just returned to torch's caching allocator (no new device mapping)
        sell = C.c_size_t()
        nat.check(lib.aqp_problem_sell_bytes(h, C.byref(sell)), "aqp_problem_sell_bytes")
        self.sell = None
        # AQP_NO_SELL_ATTACH=1 (test hook): leave the SELL copies unattached, as
        # a C-ABI caller may -- the CSR plans (incl. a deferred A' plan) serve
        if sell.value and os.environ.get("AQP_NO_SELL_ATTACH", "") != "1":
            self.sell = self.ctx.empty(sell.value)
            nat.check(lib.aqp_problem_attach_sell(h, C.c_void_p(self.sell.data_ptr()), sell.value),
                      "aqp_problem_attach_sell")
        if phases:
            self.ctx.torch.cuda.synchronize()
            self.timing["create"] = time.perf_counter() - t_up
        self.handle = h
        self.n, self.m = p.n, p.m
        self.kind = q.kind
        self.persistent_bytes = int(pb.value)
        self.part = part
        if part is None:
            self.rank, self.nranks = 0, 1
            self.rows = (0, p.n, 0, p.m)
            self.plans = None
        else:
            self.rank, self.nranks = part.rank, part.me.nranks
            self.rows = (part.me.n0, part.me.n1, part.me.m0, part.me.m1)
            self.plans = part.plans
        info = nat.ProblemInfo()
        nat.check(lib.aqp_problem_get_info(h, C.byref(info)))
        self.info = info

    def setup_info(self) -> nat.SetupInfo:
        """Validation flags and setup scalars computed on the device
        (aqp_problem_setup_info: validate / inf_norm_bound / diag_bound /
        finite_bound_scale / |c|_inf of the reference's solve entry)."""
        info = nat.SetupInfo()
        nat.check(self.ctx.lib.aqp_problem_setup_info(self.handle, C.byref(info)), "aqp_problem_setup_info")
        return info

    def scale(self, ruiz_iters: int = 10, pock_chambolle: bool = False):
        """Equilibrate this device problem in place (aqp_problem_scale); returns
        the (D, E) scalings as device tensors (x = D x~, y = E y~)."""
        torch = self.ctx.torch
        dev = f"cuda:{self.ctx.device}"
        D = torch.empty(max(self.n, 1), dtype=torch.float64, device=dev)
        E = torch.empty(max(self.m, 1), dtype=torch.float64, device=dev)
        scratch = torch.empty(2 * self.n + self.m + 1, dtype=torch.float64, device=dev)
        nat.check(self.ctx.lib.aqp_problem_scale(self.handle, int(ruiz_iters), int(bool(pock_chambolle)),
                                                 C.c_void_p(D.data_ptr()), C.c_void_p(E.data_ptr()),
                                                 C.c_void_p(scratch.data_ptr()), scratch.numel() * 8),
                  "aqp_problem_scale")
        return D[: self.n], E[: self.m]

    def close(self):
        if getattr(self, "handle", None):
            self.ctx.lib.aqp_problem_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceSolver:
    """Iteration state of one solve (engine.py:125-155 plus the locals of solve)."""

    X_EVAL, Y, DUAL_SLACK, YRAY0, YRAY1, XRAY0, XRAY1, X = range(8)

    def __init__(self, prob: DeviceProblem, *, eps_tol, eps_inf, gamma_sys, tol_scale, tol_floor, diag_bound,
                 adaptive, max_inner, halpern):
        self.prob = prob
        self.lib = prob.ctx.lib
        prm = nat.SolverParamsC()
        prm.eps_tol, prm.eps_inf, prm.gamma_sys = eps_tol, eps_inf, gamma_sys
        prm.tol_scale, prm.tol_floor, prm.diag_bound = tol_scale, tol_floor, diag_bound
        prm.adaptive, prm.max_inner, prm.halpern = int(adaptive), int(max_inner), int(halpern)
        sz = C.c_size_t()
        nat.check(self.lib.aqp_solver_sizes(prob.handle, C.byref(sz)), "aqp_solver_sizes")
        self.workspace = prob.ctx.empty(sz.value)
        h = C.c_void_p()
        nat.check(self.lib.aqp_solver_create(prob.handle, C.byref(prm), C.c_void_p(self.workspace.data_ptr()),
                                             sz.value, C.byref(h)), "aqp_solver_create")
        self.handle = h
        self.sc = nat.Scalars()

    # -- scalars ----------------------------------------------------------
    def init(self, sc: nat.Scalars):
        nat.check(self.lib.aqp_solver_init(self.handle, C.byref(sc)), "aqp_solver_init")

    def get_scalars(self) -> nat.Scalars:
        sc = nat.Scalars()
        nat.check(self.lib.aqp_solver_get_scalars(self.handle, C.byref(sc)), "aqp_solver_get_scalars")
        return sc

    def set_scalars(self, sc: nat.Scalars):
        nat.check(self.lib.aqp_solver_set_scalars(self.handle, C.byref(sc)), "aqp_solver_set_scalars")

    # -- work ----------------------------------------------------------------
    def estimate_norm(self, v0: np.ndarray, iters: int):
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        out = C.c_double()
        ann = C.c_int()
        nat.check(self.lib.aqp_solver_estimate_norm(self.handle, v0.ctypes.data, int(iters), C.byref(out),
                                                    C.byref(ann)), "aqp_solver_estimate_norm")
        return out.value, bool(ann.value)

    def run(self, n_iters: int):
        nat.check(self.lib.aqp_solver_run(self.handle, int(n_iters)), "aqp_solver_run")

    def check(self, with_rays: bool) -> nat.CheckResult:
        cr = nat.CheckResult()
        nat.check(self.lib.aqp_solver_check(self.handle, int(bool(with_rays)), C.byref(cr)), "aqp_solver_check")
        return cr

    def mark_cert(self):
        nat.check(self.lib.aqp_solver_mark_cert(self.handle))

    def restart(self):
        nat.check(self.lib.aqp_solver_restart(self.handle))

    def rollback(self):
        nat.check(self.lib.aqp_solver_rollback(self.handle))

    def reset_window(self):
        nat.check(self.lib.aqp_solver_reset_window(self.handle))

    def _length(self, which: int) -> int:
        n0, n1, m0, m1 = self.prob.rows
        return m1 - m0 if which in (self.Y, self.YRAY0, self.YRAY1) else n1 - n0

    def prefault(self, whiches) -> None:
        """Allocate and page in the host buffers of coming reads (the result
        vectors) on a background thread while the solve loop runs on the
        device: a fresh 400 MB numpy array otherwise takes its page faults
        inside the timed read-back."""
        import threading

        spare = {}

        def work():
            for w in whiches:
                a = np.empty(self._length(w), dtype=np.float64)
                a[::512] = 0.0  # one write per 4 KB page
                spare[w] = a

        self._spare = spare
        self._prefault = threading.Thread(target=work, daemon=True)
        self._prefault.start()

    def read(self, which: int) -> np.ndarray:
        """The whole vector, or (row shard) this rank's slice of it."""
        length = self._length(which)
        out = None
        pf = getattr(self, "_prefault", None)
        if pf is not None and not pf.is_alive():  # never wait for it
            out = self._spare.pop(which, None)
        if out is None:
            out = np.empty(length, dtype=np.float64)
        nat.check(self.lib.aqp_solver_read(self.handle, int(which), out.ctypes.data, length), "aqp_solver_read")
        return out

    def time_kernel(self, kernel: int, reps: int, flush=None) -> float:
        """Average device ms of one stand-alone launch of a hot kernel (see aqp.h)."""
        out = C.c_double()
        fptr = C.c_void_p(flush.data_ptr()) if flush is not None else None
        fbytes = flush.numel() * flush.element_size() if flush is not None else 0
        nat.check(self.lib.aqp_solver_time_kernel(self.handle, int(kernel), int(reps), fptr, fbytes, C.byref(out)),
                  "aqp_solver_time_kernel")
        return out.value

    def trace(self, cap: int = 1 << 20) -> np.ndarray:
        """(tag, ns) stamps recorded since the last call (AQP_TRACE=1), as an (k, 2) uint64 array."""
        buf = np.empty(2 * cap, dtype=np.uint64)
        cnt = C.c_int64()
        nat.check(self.lib.aqp_solver_trace(self.handle, buf.ctypes.data, cap, C.byref(cnt)), "aqp_solver_trace")
        return buf[: 2 * cnt.value].reshape(-1, 2)

    def counters(self):
        buf = (C.c_int64 * 3)()
        nat.check(self.lib.aqp_solver_counters(self.handle, buf))
        return int(buf[0]), int(buf[1])

    def uses_pdl(self) -> bool:
        buf = (C.c_int64 * 3)()
        nat.check(self.lib.aqp_solver_counters(self.handle, buf))
        return bool(buf[2])

    def import_scaled(self, src: "DeviceSolver", D, E):
        """This (original-problem) solver <- src's iterate, anchor and window
        sums mapped back from the scaled space (aqp_solver_import_scaled)."""
        nat.check(self.lib.aqp_solver_import_scaled(self.handle, src.handle, C.c_void_p(D.data_ptr()),
                                                    C.c_void_p(E.data_ptr())), "aqp_solver_import_scaled")

    # -- row shards -------------------------------------------------------------
    def exchange_region(self):
        """(device address, bytes) of the peer-written front of the workspace."""
        base, nbytes = C.c_void_p(), C.c_size_t()
        nat.check(self.lib.aqp_solver_exchange_region(self.handle, C.byref(base), C.byref(nbytes)))
        return int(base.value), int(nbytes.value)

    def set_halos(self, x_ranges, y_ranges):
        """Per-rank gather ranges [lo, hi) for the x and y sides (aqp_solver_set_halos)."""
        xr = np.ascontiguousarray(np.asarray(x_ranges, dtype=np.int64).reshape(-1))
        yr = np.ascontiguousarray(np.asarray(y_ranges, dtype=np.int64).reshape(-1))
        nat.check(self.lib.aqp_solver_set_halos(self.handle, xr.ctypes.data_as(nat.c_int64_p),
                                                yr.ctypes.data_as(nat.c_int64_p), len(xr) // 2),
                  "aqp_solver_set_halos")

    def connect(self, peer_bases):
        """Bind the peers' workspace mappings (index = rank) and build the graph."""
        arr = (C.c_void_p * len(peer_bases))(*[C.c_void_p(int(b)) for b in peer_bases])
        nat.check(self.lib.aqp_solver_connect(self.handle, arr, len(peer_bases)), "aqp_solver_connect")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.aqp_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
