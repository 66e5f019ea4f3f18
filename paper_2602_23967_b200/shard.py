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
import dataclasses
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


def _counts(problem):
    """Column counts of A and of Q's upper triangle (one bincount each over the
    nonzeros -- the only O(nnz) host passes of the plan), cached on the
    problem object: every rank of a process group plans the same problem."""
    cached = getattr(problem, "_aqp_shard_counts", None)
    if cached is not None:
        return cached
    a = problem.constraint_matrix
    n = problem.n
    acol = np.bincount(np.asarray(a.indices), minlength=n) if a.nnz else np.zeros(n, dtype=np.int64)
    q = problem.quad
    pq = q if q.kind == "sparse" else (q.p if q.kind == "sparse_low_rank" else None)
    qcol = None
    if pq is not None:
        qi = np.asarray(pq.upper.indices)
        qcol = np.bincount(qi, minlength=n) if len(qi) else np.zeros(n, dtype=np.int64)
    out = (acol, qcol)
    try:
        object.__setattr__(problem, "_aqp_shard_counts", out)
    except Exception:
        pass
    return out


def partition(problem, nranks: int) -> List[Rows]:
    """Contiguous row blocks per rank, balanced by per-iteration bytes.

    y side: rows of A (nnz per row); x side: rows of A' (column counts of A)
    plus rows of the full symmetric Q (upper-row + upper-column counts)."""
    if not 1 <= nranks <= 8:
        raise ValueError("row shards support 1..8 ranks")
    a = problem.constraint_matrix
    wy = _Y_ROW_BYTES + _NNZ_BYTES * np.diff(np.asarray(a.indptr)).astype(np.float64)
    acol, qcol = _counts(problem)
    wx = _X_ROW_BYTES + _NNZ_BYTES * acol.astype(np.float64)
    q = problem.quad
    if q.kind == "sparse":
        rc = np.diff(np.asarray(q.upper.indptr)).astype(np.float64)
        wx = wx + _NNZ_BYTES * (rc + qcol.astype(np.float64))
    cx, cy = _split(wx, nranks), _split(wy, nranks)
    return [(cx[k], cx[k + 1], cy[k], cy[k + 1]) for k in range(nranks)]


@dataclasses.dataclass(frozen=True)
class RankPlan:
    """What rank `rank` stores and gathers (aqp_shard_desc).

    * rows [n0, n1) of A' and of the full symmetric Q, rows [m0, m1) of A;
    * the uploaded A block = rows ``ywin`` of A (the rank's own rows plus every
      row with a nonzero in columns [n0, n1), i.e. the sources of its A'
      rows), from which the device keeps rows [m0, m1) and builds A' rows
      [n0, n1);
    * the uploaded P block = upper-triangle rows [q_row0, n1) (its own rows
      plus every row j < n0 with an upper entry in columns [n0, n1), the
      sources of the mirrored lower part);
    * gather halos ``xhalo`` (columns of its rows of A and Q) and ``yhalo``
      (columns of its rows of A'), and the windows ``xwin`` / ``ywin`` =
      halo hull its own rows: the only entries of x / y it ever holds.
    """

    rank: int
    nranks: int
    n0: int
    n1: int
    m0: int
    m1: int
    q_row0: int
    xhalo: Tuple[int, int]
    yhalo: Tuple[int, int]
    xwin: Tuple[int, int]
    ywin: Tuple[int, int]
    a_local_nnz: int
    at_local_nnz: int
    q_local_nnz: int


def _row_extents(indptr: np.ndarray, indices: np.ndarray, ncols: int):
    """First / last column of every CSR row (sorted rows); empty rows: (ncols, -1)."""
    indptr = np.asarray(indptr)
    nz = np.diff(indptr) > 0
    lo = np.full(len(indptr) - 1, ncols, dtype=np.int64)
    hi = np.full(len(indptr) - 1, -1, dtype=np.int64)
    idx = np.asarray(indices)
    lo[nz] = idx[indptr[:-1][nz]]
    hi[nz] = idx[indptr[1:][nz] - 1]
    return lo, hi


def _hull(*ranges) -> Tuple[int, int]:
    rs = [(int(a), int(b)) for a, b in ranges if b > a]
    if not rs:
        return (0, 0)
    return (min(a for a, _ in rs), max(b for _, b in rs))


def plan(problem, nranks: int, parts: Optional[Sequence[Rows]] = None) -> List[RankPlan]:
    """Row partition plus, per rank, the blocks it uploads, its gather halos
    and windows.  O(n + m) plus two bincounts over the nonzeros; every rank
    computes the identical plan from the same problem."""
    parts = list(parts) if parts is not None else partition(problem, nranks)
    a = problem.constraint_matrix
    n, m = problem.n, problem.m
    ip, ix = np.asarray(a.indptr), np.asarray(a.indices)
    alo, ahi = _row_extents(ip, ix, n)
    colcnt, qcol = _counts(problem)
    ccum = np.concatenate([[0], np.cumsum(colcnt)])
    q = problem.quad
    pq = q if q.kind == "sparse" else (q.p if q.kind == "sparse_low_rank" else None)
    if pq is not None:
        up = pq.upper
        qp, qi = np.asarray(up.indptr), np.asarray(up.indices)
        qlo, qhi = _row_extents(qp, qi, n)
        # full row i of Q = upper row i + mirrored off-diagonal upper entries (j, i):
        # column i's upper count minus its diagonal (the first entry of a row
        # that stores it -- upper rows are sorted)
        has_diag = (qlo == np.arange(n)).astype(np.int64)
        fullcnt = np.diff(qp) + qcol - has_diag
        fcum = np.concatenate([[0], np.cumsum(fullcnt)])
    out = []
    for r, (n0, n1, m0, m1) in enumerate(parts):
        xr = [(int(alo[m0:m1].min(initial=n)), int(ahi[m0:m1].max(initial=-1)) + 1)]
        q_row0 = n0
        qloc = 0
        if pq is not None:
            xr.append((n0, int(qhi[n0:n1].max(initial=-1)) + 1))  # upper part: j >= i
            src = np.flatnonzero((qhi[:n0] >= n0) & (qlo[:n0] < n1))  # mirrored part: rows j < n0
            if src.size:
                q_row0 = int(src[0])
                xr.append((q_row0, n0))
            qloc = int(fcum[n1] - fcum[n0])
        xhalo = _hull(*xr)
        yrows = np.flatnonzero((alo < n1) & (ahi >= n0))  # rows of A with a nonzero in columns [n0, n1)
        yhalo = (int(yrows[0]), int(yrows[-1]) + 1) if yrows.size else (0, 0)
        out.append(RankPlan(rank=r, nranks=nranks, n0=n0, n1=n1, m0=m0, m1=m1, q_row0=q_row0,
                            xhalo=xhalo, yhalo=yhalo, xwin=_hull(xhalo, (n0, n1)), ywin=_hull(yhalo, (m0, m1)),
                            a_local_nnz=int(ip[m1] - ip[m0]), at_local_nnz=int(ccum[n1] - ccum[n0]),
                            q_local_nnz=qloc))
    return out


@dataclasses.dataclass
class LocalPart:
    """Host views of one rank's blocks (inputs of aqp_problem_create with a
    shard descriptor) plus the plan of every rank."""

    plans: List[RankPlan]
    rank: int
    a_indptr: np.ndarray
    a_indices: np.ndarray
    a_data: np.ndarray
    q_indptr: Optional[np.ndarray]
    q_indices: Optional[np.ndarray]
    q_data: Optional[np.ndarray]
    q_vec: Optional[np.ndarray]       # DiagonalQuad values or P's diagonal, entries [n0, n1)
    r_indptr: Optional[np.ndarray]
    r_indices: Optional[np.ndarray]
    r_data: Optional[np.ndarray]
    r_dense: bool
    cost: np.ndarray
    var_lo: np.ndarray
    var_hi: np.ndarray
    con_lo: np.ndarray
    con_hi: np.ndarray

    @property
    def me(self) -> RankPlan:
        return self.plans[self.rank]


def _block(indptr, indices, data, r0, r1):
    indptr = np.asarray(indptr)
    k0, k1 = int(indptr[r0]), int(indptr[r1])
    return indptr[r0:r1 + 1] - k0, np.asarray(indices)[k0:k1], np.asarray(data)[k0:k1]


def local_part(problem, plans: List[RankPlan], rank: int) -> LocalPart:
    """This rank's blocks as host views (no copies of the big arrays)."""
    me = plans[rank]
    n0, n1, m0, m1 = me.n0, me.n1, me.m0, me.m1
    a = problem.constraint_matrix
    ai, ax, ad = _block(a.indptr, a.indices, a.data, me.ywin[0], me.ywin[1])
    q = problem.quad
    qi = qx = qd = qv = None
    ri = rx = rd = None
    dense = False
    if q.kind == "diagonal":
        qv = np.asarray(q.values)[n0:n1]
    else:
        pq = q if q.kind == "sparse" else q.p
        qi, qx, qd = _block(pq.upper.indptr, pq.upper.indices, pq.upper.data, me.q_row0, n1)
        qv = np.asarray(pq.diag)[n0:n1]
        if q.kind == "sparse_low_rank":
            from .device import _full_rows

            r = q.r
            nl = n1 - n0
            if _full_rows(r):  # dense factor: columns [n0, n1) of every row, row-major
                dense = True
                rd = np.ascontiguousarray(np.asarray(r.data).reshape(r.rows, r.cols)[:, n0:n1]).reshape(-1)
                ri = np.arange(r.rows + 1, dtype=np.int64) * nl
                rx = None
            else:
                rp, rc, rv = np.asarray(r.indptr), np.asarray(r.indices), np.asarray(r.data)
                keep = (rc >= n0) & (rc < n1)
                rows = np.repeat(np.arange(r.rows), np.diff(rp))
                ri = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=r.rows))]).astype(np.int64)
                rx, rd = rc[keep], rv[keep]
    return LocalPart(plans=plans, rank=rank, a_indptr=ai, a_indices=ax, a_data=ad, q_indptr=qi, q_indices=qx,
                     q_data=qd, q_vec=qv, r_indptr=ri, r_indices=rx, r_data=rd, r_dense=dense,
                     cost=np.asarray(problem.cost)[n0:n1], var_lo=np.asarray(problem.var_bounds.lower)[n0:n1],
                     var_hi=np.asarray(problem.var_bounds.upper)[n0:n1],
                     con_lo=np.asarray(problem.con_bounds.lower)[m0:m1],
                     con_hi=np.asarray(problem.con_bounds.upper)[m0:m1])


def halos(problem, parts: Sequence[Rows]):
    """Gather halos per rank (see RankPlan): two lists of [lo, hi) ranges."""
    pl = plan(problem, len(parts), parts)
    return [p.xhalo for p in pl], [p.yhalo for p in pl]


def _set_halos(solver):
    plans = solver.prob.plans
    solver.set_halos([p.xhalo for p in plans], [p.yhalo for p in plans])


_Handle = C.c_char * 64  # cudaIpcMemHandle_t


class PeerGroup:
    """What a sharded solve needs from its peers (see module docstring)."""

    rank: int = 0
    nranks: int = 1

    def connect(self, solver) -> None:  # pragma: no cover - interface
        raise NotImplementedError

    def agree_any(self, flag: bool) -> bool:  # pragma: no cover - interface
        raise NotImplementedError

    def gather(self, arr: np.ndarray) -> List[np.ndarray]:  # pragma: no cover - interface
        """Every rank's `arr`, in rank order (host arrays; collective)."""
        raise NotImplementedError

    def concat(self, arr: np.ndarray) -> np.ndarray:
        """The ranks' row slices joined into the whole vector (collective)."""
        return np.concatenate(self.gather(np.ascontiguousarray(arr)))

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
        _set_halos(solver)
        solver.connect(bases)
        self.dist.barrier(group=self.group)

    def agree_any(self, flag: bool) -> bool:
        import torch

        t = torch.tensor([1 if flag else 0], dtype=torch.int32)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(int(t.item()))

    def gather(self, arr: np.ndarray) -> List[np.ndarray]:
        out = [None] * self.nranks
        self.dist.all_gather_object(out, arr, group=self.group)
        return out

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
        self.items: List = [None] * nranks


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
        _set_halos(solver)
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

    def gather(self, arr: np.ndarray) -> List[np.ndarray]:
        sh = self.shared
        sh.items[self.rank] = arr
        sh.barrier.wait()
        out = list(sh.items)
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
            from .batch import pooled_stream

            torch.cuda.set_device(device)
            with torch.cuda.stream(pooled_stream(device, 1000 + r)):  # one cached stream per virtual rank
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


__all__ = ["partition", "plan", "local_part", "halos", "RankPlan", "LocalPart", "PeerGroup", "DistGroup",
           "LocalGroup", "solve_local", "rows_of"]
