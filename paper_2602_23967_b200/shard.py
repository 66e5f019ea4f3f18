"""Row-sharded solves across GPUs.

The reference has no multi-GPU path (its only parallelism is a process pool
over independent instances, ``anchorqp/bench.py:89-98``); this module adds the
row partition that BASELINE.json's north star asks for on instances like C5:

* rank r owns a contiguous block of rows of A (the y side, ``[m0, m1)``) and
  of A' and Q (the x side, ``[n0, n1)``), balanced by the bytes each row moves
  per iteration (nonzeros + vector entries);
* every vector an SpMV gathers (y, x0/x_t, xbar, x_eval, ray candidates) is
  kept whole on every rank; the kernel that produces a rank's slice also
  stores it into the peers' copies over NVLink (P2P stores into CUDA-IPC
  mapped workspaces), and one-block mailbox exchanges combine every reduction
  in rank order -- so all ranks hold identical scalars and take identical
  branches, inside the same CUDA graph, with no NCCL call on the data path;
* ``torch.distributed`` (NCCL or gloo) is only plumbing: it exchanges the IPC
  handles and makes the host-side decisions that read a clock (time limit)
  collective.

Two peer groups drive the same kernels:

* :class:`DistGroup` -- one process per GPU (``torchrun``), CUDA IPC.
* :class:`LocalGroup` -- ``nranks`` virtual ranks on ONE device in one
  process (one thread + stream each; peer stores are local stores).  It runs
  the exact multi-GPU code path (partition, peer stores, exchanges, graph
  barriers) and is how the path is parity-tested on a single B200.
"""

from __future__ import annotations

import ctypes as C
import threading
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .errors import DeviceError

Rows = Tuple[int, int, int, int]  # n0, n1, m0, m1

# bytes a row moves per outer iteration besides its nonzeros (SURVEY.md §8(d):
# ~88-112 B per x entry, ~64 B per y entry) and per nonzero (12 B per pass)
_X_ROW_BYTES, _Y_ROW_BYTES, _NNZ_BYTES = 112.0, 64.0, 12.0


def _split(weights: np.ndarray, parts: int) -> List[int]:
    """Cut points 0 = c0 < c1 < ... < c_parts = len(weights) with about equal
    weight per part and at least one row per part."""
    n = len(weights)
    if n < parts:
        raise ValueError(f"{n} rows cannot be split over {parts} ranks")
    cum = np.concatenate([[0.0], np.cumsum(weights, dtype=np.float64)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, parts):
        c = int(np.searchsorted(cum, total * k / parts, side="left"))
        c = max(c, cuts[-1] + 1)
        c = min(c, n - (parts - k))
        cuts.append(c)
    cuts.append(n)
    return cuts


def partition(problem, nranks: int) -> List[Rows]:
    """Contiguous row blocks per rank, balanced by per-iteration bytes.

    y side: rows of A (nnz per row); x side: rows of A' (column counts of A)
    plus rows of the full symmetric Q (upper-row + upper-column counts)."""
    if not 1 <= nranks <= 8:
        raise ValueError("row shards support 1..8 ranks")
    a = problem.constraint_matrix
    n, m = problem.n, problem.m
    wy = _Y_ROW_BYTES + _NNZ_BYTES * np.diff(np.asarray(a.indptr)).astype(np.float64)
    colcnt = np.bincount(np.asarray(a.indices), minlength=n).astype(np.float64)
    wx = _X_ROW_BYTES + _NNZ_BYTES * colcnt
    q = problem.quad
    if q.kind == "sparse":
        up = q.upper
        rc = np.diff(np.asarray(up.indptr)).astype(np.float64)
        cc = np.bincount(np.asarray(up.indices), minlength=n).astype(np.float64)
        wx = wx + _NNZ_BYTES * (rc + cc)
    cx, cy = _split(wx, nranks), _split(wy, nranks)
    return [(cx[k], cx[k + 1], cy[k], cy[k + 1]) for k in range(nranks)]


def halos(problem, parts: Sequence[Rows]):
    """Gather halos per rank: rank k gathers x only at the columns of its rows
    of A and of the full symmetric Q, and y only at the columns of its rows of
    A' (= the rows of A having a nonzero in its columns).  Returns two lists of
    [lo, hi) ranges (global indices; empty ranges as (0, 0))."""
    a = problem.constraint_matrix
    n, m = problem.n, problem.m
    ip, ix = np.asarray(a.indptr), np.asarray(a.indices)
    arow = np.repeat(np.arange(m), np.diff(ip))
    q = problem.quad
    if q.kind == "sparse":
        up = q.upper
        qp, qi = np.asarray(up.indptr), np.asarray(up.indices)
        qrow = np.repeat(np.arange(n), np.diff(qp))
    xr, yr = [], []
    for n0, n1, m0, m1 in parts:
        lo, hi = n, 0
        cols = ix[ip[m0]:ip[m1]]                      # A rows [m0, m1)
        if cols.size:
            lo, hi = min(lo, int(cols.min())), max(hi, int(cols.max()) + 1)
        if q.kind == "sparse":
            ucols = qi[qp[n0]:qp[n1]]                  # upper rows [n0, n1): j >= i
            if ucols.size:
                lo, hi = min(lo, int(ucols.min())), max(hi, int(ucols.max()) + 1)
            sel = (qi >= n0) & (qi < n1)               # mirrored lower part: rows j < i
            if sel.any():
                r = qrow[sel]
                lo, hi = min(lo, int(r.min())), max(hi, int(r.max()) + 1)
        xr.append((lo, hi) if hi > lo else (0, 0))
        sel = (ix >= n0) & (ix < n1)                   # A' rows [n0, n1) = A's columns
        if sel.any():
            r = arow[sel]
            yr.append((int(r.min()), int(r.max()) + 1))
        else:
            yr.append((0, 0))
    return xr, yr


def _set_halos(solver, problem, nranks):
    parts = partition(problem, nranks)
    xr, yr = halos(problem, parts)
    solver.set_halos(xr, yr)


_Handle = C.c_char * 64  # cudaIpcMemHandle_t


class PeerGroup:
    """What a sharded solve needs from its peers (see module docstring)."""

    rank: int = 0
    nranks: int = 1

    def connect(self, solver) -> None:  # pragma: no cover - interface
        raise NotImplementedError

    def agree_any(self, flag: bool) -> bool:  # pragma: no cover - interface
        raise NotImplementedError

    def close(self) -> None:
        pass


class DistGroup(PeerGroup):
    """One process per GPU under ``torch.distributed`` (torchrun); the peers'
    solver workspaces are mapped with CUDA IPC (NVLink P2P on one node)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise DeviceError("DistGroup needs torch.distributed initialised (torchrun)")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self._mapped: List[Tuple[int, int]] = []

    def connect(self, solver) -> None:
        lib = nat.load()
        base, _ = solver.exchange_region()
        handle = _Handle()
        off = C.c_size_t()
        nat.check(lib.aqp_ipc_get_handle(C.c_void_p(base), handle, C.byref(off)), "aqp_ipc_get_handle")
        mine = (bytes(handle), int(off.value))
        everyone = [None] * self.nranks
        self.dist.all_gather_object(everyone, mine, group=self.group)
        bases = []
        for k, (h, o) in enumerate(everyone):
            if k == self.rank:
                bases.append(base)
                continue
            hb = _Handle.from_buffer_copy(h)
            ptr = C.c_void_p()
            nat.check(lib.aqp_ipc_open(hb, o, C.byref(ptr)), "aqp_ipc_open")
            self._mapped.append((int(ptr.value), o))
            bases.append(int(ptr.value))
        self.dist.barrier(group=self.group)  # every rank's mailbox is zero before anyone writes
        if getattr(solver, "problem_host", None) is not None:
            _set_halos(solver, solver.problem_host, self.nranks)
        solver.connect(bases)
        self.dist.barrier(group=self.group)

    def agree_any(self, flag: bool) -> bool:
        import torch

        t = torch.tensor([1 if flag else 0], dtype=torch.int32)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(int(t.item()))

    def close(self) -> None:
        lib = nat.load()
        for ptr, off in self._mapped:
            lib.aqp_ipc_close(C.c_void_p(ptr), off)
        self._mapped = []


class _LocalShared:
    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.bases: List[Optional[int]] = [None] * nranks
        self.flags = [False] * nranks


class LocalGroup(PeerGroup):
    """Virtual rank `rank` of `nranks` sharing one device in one process."""

    def __init__(self, shared: _LocalShared, rank: int):
        self.shared = shared
        self.rank = rank
        self.nranks = shared.nranks

    @staticmethod
    def create(nranks: int) -> List["LocalGroup"]:
        sh = _LocalShared(nranks)
        return [LocalGroup(sh, r) for r in range(nranks)]

    def connect(self, solver) -> None:
        base, _ = solver.exchange_region()
        self.shared.bases[self.rank] = base
        self.shared.barrier.wait()  # all created (mailboxes zeroed) and published
        if getattr(solver, "problem_host", None) is not None:
            _set_halos(solver, solver.problem_host, self.nranks)
        solver.connect(list(self.shared.bases))
        # graph instantiation may synchronise the device: no rank may start
        # exchanging (spinning) while another rank still builds its graph
        self.shared.barrier.wait()

    def agree_any(self, flag: bool) -> bool:
        sh = self.shared
        sh.flags[self.rank] = bool(flag)
        sh.barrier.wait()
        out = any(sh.flags)
        sh.barrier.wait()
        return out


def solve_local(problem, params=None, nranks: int = 2, device: int = 0, timeout: float = 3600.0, **kw):
    """Row-sharded solve over `nranks` virtual ranks on one device (threads,
    one CUDA stream each).  Returns the per-rank SolveResults (identical
    status / counts / vectors on every rank).

    The ranks' exchange kernels spin on each other, so their streams must sit
    on distinct hardware queues: run with CUDA_DEVICE_MAX_CONNECTIONS=32 set
    before CUDA initialises (tests/conftest.py does).  A violated assumption
    surfaces as an exchange-timeout DeviceError, never as a hang."""
    import torch

    from .engine import solve

    groups = LocalGroup.create(nranks)
    results: List = [None] * nranks
    errors: List = [None] * nranks

    def work(r):
        try:
            torch.cuda.set_device(device)
            with torch.cuda.stream(torch.cuda.Stream(device)):
                results[r] = solve(problem, params, device=device, group=groups[r], **kw)
        except BaseException as exc:  # reported after join
            errors[r] = exc
            try:
                groups[r].shared.barrier.abort()
            except Exception:
                pass

    threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(nranks)]
    for t in threads:
        t.start()
    import time as _time

    deadline = _time.monotonic() + timeout
    for t in threads:
        t.join(max(0.0, deadline - _time.monotonic()))
    if any(t.is_alive() for t in threads):
        import sys
        import traceback

        frames = sys._current_frames()
        dump = []
        for r, t in enumerate(threads):
            if t.is_alive() and t.ident in frames:
                dump.append(f"rank {r}:\n" + "".join(traceback.format_stack(frames[t.ident])))
        errs = [f"rank {r}: {e!r}" for r, e in enumerate(errors) if e is not None]
        raise DeviceError("sharded local solve did not finish (a rank is stuck)\n" + "\n".join(errs + dump))
    errs = [(r, e) for r, e in enumerate(errors) if e is not None]
    if len(errs) == 1:
        raise errs[0][1]
    if errs:
        raise DeviceError("sharded local solve failed on ranks " + "; ".join(f"{r}: {e!r}" for r, e in errs))
    return results


def rows_of(problem, group: PeerGroup) -> Rows:
    return partition(problem, group.nranks)[group.rank]


__all__ = ["partition", "halos", "PeerGroup", "DistGroup", "LocalGroup", "solve_local", "rows_of"]
