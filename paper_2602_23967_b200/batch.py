"""Many-instance batching on one B200 and the benchmark records of the
reference harness (reference ``aq/bench.py``).

The reference's only data-parallel strategy is a process pool over instances
(``aq/bench.py:89-98``).  A single C1- or C4-sized solve cannot fill a B200:
its SpMV passes are a few dozen blocks and every window ends in a host
round trip.  :func:`solve_many` therefore runs ``streams`` solves at once, one
host thread and one CUDA stream each, so the device interleaves the kernels
of independent solves (each solve's window is still one CUDA graph).  Across
the GPUs of a node, run one process per GPU and give each a stride of the
instances (:func:`shard_instances`).

``RunRecord``, :func:`sgm10`, :func:`summarize` and :func:`run_benchmark` keep
the reference's fields and arithmetic (``aq/bench.py:18-113``).
"""

from __future__ import annotations

import dataclasses
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from typing import Iterable, List, Optional, Sequence

import numpy as np

from .engine import SolveStatus, SolverParams, solve
from .errors import EmptyInput, ParseError


@dataclasses.dataclass(frozen=True)
class RunRecord:
    """One instance's outcome (reference ``aq/bench.py:18-36``)."""

    instance: str
    status: str
    outer_iterations: int
    inner_iterations: int
    seconds: float
    r_primal: float
    r_dual: float
    r_gap: float
    objective: float

    @property
    def solved(self) -> bool:
        return self.status == SolveStatus.OPTIMAL.value

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)


def sgm10(times, limit: float, solved_mask) -> float:
    """Shifted geometric mean, shift 10; unsolved entries are charged the time
    limit (reference ``aq/bench.py:39-50``)."""
    t = np.asarray(times, dtype=np.float64)
    ok = np.asarray(solved_mask, dtype=bool)
    if t.size == 0:
        raise EmptyInput("sgm10 needs at least one time")
    return float(np.exp(np.mean(np.log(np.where(ok, t, limit) + 10.0))) - 10.0)


def summarize(records: Sequence[RunRecord], time_limit: float) -> dict:
    """Aggregate of a benchmark run (reference ``aq/bench.py:102-113``)."""
    if not records:
        raise EmptyInput("no run records to summarize")
    times = [r.seconds for r in records]
    solved = [r.solved for r in records]
    n_ok = int(sum(solved))
    return {
        "instances": len(records),
        "solved": n_ok,
        "failed": len(records) - n_ok,
        "sgm10_seconds": sgm10(times, time_limit, solved),
        "mean_seconds": float(np.mean([t if s else time_limit for t, s in zip(times, solved)])),
        "time_limit": time_limit,
    }


def record_of(name: str, result) -> RunRecord:
    rep = result.report
    return RunRecord(instance=name, status=result.status.value, outer_iterations=result.outer_iterations,
                     inner_iterations=result.inner_iterations, seconds=result.seconds, r_primal=rep.r_primal,
                     r_dual=rep.r_dual, r_gap=rep.r_gap, objective=rep.primal_objective)


_pool_lock = threading.Lock()
_stream_pool = {}  # (device, slot) -> torch stream, reused by every call


def pooled_stream(device: int, slot: int):
    """The process-wide stream of worker slot `slot` on `device`.  Solves on
    one stream share one libaqp context (and its pinned staging), so reusing
    the streams across calls bounds the contexts -- and the pinned host
    memory -- to one per slot instead of one per call."""
    import torch

    with _pool_lock:
        s = _stream_pool.get((device, slot))
        if s is None:
            s = _stream_pool[(device, slot)] = torch.cuda.Stream(device)
        return s


def solve_many(problems: Sequence, params: Optional[SolverParams] = None, streams: int = 8, device: int = 0,
               progress=None) -> List:
    """Solve independent instances concurrently on one device.

    ``streams`` host threads each own a CUDA stream and run whole solves
    (problem upload, window graphs, checks) one after another; results come
    back in input order.  Each result is exactly what :func:`solve` returns
    for that instance alone (the solves share nothing but the device)."""
    import torch

    probs = list(problems)
    if not probs:
        return []
    streams = max(1, min(int(streams), len(probs)))
    if streams == 1:
        return [solve(p, params, progress, device=device) for p in probs]

    import queue

    slots = queue.Queue()
    for i in range(streams):
        slots.put(i)

    def one(p):
        slot = slots.get()  # a stream no other worker is using right now
        try:
            torch.cuda.set_device(device)
            with torch.cuda.stream(pooled_stream(device, slot)):
                r = solve(p, params, progress, device=device)
                torch.cuda.current_stream().synchronize()
                return r
        finally:
            slots.put(slot)

    with ThreadPoolExecutor(max_workers=streams) as pool:
        return list(pool.map(one, probs))


def shard_instances(items: Sequence, rank: int, world: int) -> list:
    """Instances rank `rank` of `world` processes (one per GPU) takes: a stride."""
    return list(items)[rank::world]


def run_benchmark(instances: Iterable, params: SolverParams, streams: int = 8, device: int = 0,
                  names: Optional[Sequence[str]] = None) -> List[RunRecord]:
    """Solve every instance (QpProblem objects or file paths) and return the
    records sorted by instance name (reference ``aq/bench.py:89-99``)."""
    from . import io as aqio

    items = list(instances)
    probs, labels, bad = [], [], []
    for i, it in enumerate(items):
        label = names[i] if names is not None else (
            os.path.basename(os.fspath(it)) if isinstance(it, (str, os.PathLike)) else getattr(it, "name", f"#{i}"))
        if isinstance(it, (str, os.PathLike)):
            try:
                it = aqio.load_problem(it)
            except (ParseError, OSError, ValueError) as exc:  # as aq/bench.py:81-85
                bad.append(RunRecord(label, f"error: {exc}", 0, 0, 0.0, np.nan, np.nan, np.nan, np.nan))
                continue
        probs.append(it)
        labels.append(label)
    results = solve_many(probs, params, streams=streams, device=device)
    records = [record_of(n, r) for n, r in zip(labels, results)] + bad
    records.sort(key=lambda r: r.instance)
    return records


__all__ = ["RunRecord", "sgm10", "summarize", "record_of", "solve_many", "shard_instances", "run_benchmark"]
