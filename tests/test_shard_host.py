"""CPU: host side of the row-sharded path -- the row
partition, the host-level agreement of LocalGroup (threads) and DistGroup
(torch.distributed gloo, world size 2).  The device exchange itself is
covered by tests/test_gpu_shard.py."""

import os
import threading

import numpy as np
import pytest

import instances
from paper_2602_23967_b200 import shard


def _check_partition(parts, n, m):
    assert parts[0][0] == 0 and parts[-1][1] == n and parts[0][2] == 0 and parts[-1][3] == m
    for (a0, a1, b0, b1), (c0, c1, d0, d1) in zip(parts, parts[1:]):
        assert a1 == c0 and b1 == d0
    for n0, n1, m0, m1 in parts:
        assert n1 > n0 and m1 > m0


@pytest.mark.parametrize("spec", ["c1:0", "rqp:500:300:diagonal:0.02:5", "c5:5e3:50:0"])
@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_partition_covers_rows_contiguously(spec, nranks):
    p = instances.build(spec)
    parts = shard.partition(p, nranks)
    assert len(parts) == nranks
    _check_partition(parts, p.n, p.m)


def test_partition_balances_bytes():
    p = instances.build("c1:0")
    parts = shard.partition(p, 4)
    a = p.constraint_matrix
    wy = 64.0 + 12.0 * np.diff(a.indptr)
    loads = [wy[m0:m1].sum() for _, _, m0, m1 in parts]
    assert max(loads) <= 1.15 * (sum(loads) / 4)


def test_partition_edge_cases():
    assert shard._split(np.ones(8), 8) == list(range(9))
    # all the weight in one row still leaves every rank a row
    w = np.zeros(10)
    w[0] = 1e9
    cuts = shard._split(w, 4)
    assert cuts[0] == 0 and cuts[-1] == 10 and all(b > a for a, b in zip(cuts, cuts[1:]))
    with pytest.raises(ValueError):
        shard._split(np.ones(3), 4)
    with pytest.raises(ValueError):
        shard.partition(instances.build("c1:0"), 9)


def test_local_group_agree_any():
    groups = shard.LocalGroup.create(3)
    out = [None] * 3

    def work(r):
        out[r] = [groups[r].agree_any(r == 2 and k == 1) for k in range(3)]

    ts = [threading.Thread(target=work, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(30)
    assert out == [[False, True, False]] * 3


def _dist_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = shard.DistGroup()
        agreed = [g.agree_any(rank == 1 and k == 0) for k in range(2)]
        p = instances.build("c1:1")
        rows = shard.rows_of(p, g)
        joined = g.concat(np.arange(3) + 10 * rank)
        q.put((rank, agreed, rows, joined.tolist()))
    finally:
        dist.destroy_process_group()


def test_dist_group_gloo_world2():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    (r0, a0, rows0, j0), (r1, a1, rows1, j1) = res
    assert a0 == a1 == [True, False]
    assert j0 == j1 == [0, 1, 2, 10, 11, 12]
    p = instances.build("c1:1")
    assert [rows0, rows1] == shard.partition(p, 2)


@pytest.mark.parametrize("spec", ["c5:5e3:50:0", "c1:0", "rqp:500:300:diagonal:0.02:5", "c2:1e4:5e3:0"])
@pytest.mark.parametrize("nranks", [2, 5])
def test_halos_cover_every_gathered_column(spec, nranks):
    p = instances.build(spec)
    parts = shard.partition(p, nranks)
    xr, yr = shard.halos(p, parts)
    a = p.constraint_matrix.to_scipy().tocsr()
    at = a.T.tocsr()
    q = p.quad
    qf = None
    if q.kind == "sparse":
        u = q.upper.to_scipy()
        qf = (u + u.T).tocsr()
    for (n0, n1, m0, m1), (xl, xh), (yl, yh) in zip(parts, xr, yr):
        cols = [a[m0:m1].indices]
        if qf is not None:
            cols.append(qf[n0:n1].indices)
        c = np.concatenate(cols)
        assert c.size == 0 or (c.min() >= xl and c.max() < xh)
        r = at[n0:n1].indices
        assert r.size == 0 or (r.min() >= yl and r.max() < yh)


def test_banded_halos_are_strips():
    p = instances.build("c5:5e4:500:0")
    parts = shard.partition(p, 4)
    xr, yr = shard.halos(p, parts)
    for (n0, n1, m0, m1), (xl, xh) in zip(parts, xr):
        assert n0 - xl <= 1000 and xh - n1 <= 1000  # Q band (i +- 1000) dominates A's +- 500


def _full_q(p):
    q = p.quad
    pq = q if q.kind == "sparse" else (q.p if q.kind == "sparse_low_rank" else None)
    if pq is None:
        return None
    u = pq.upper.to_scipy()
    import scipy.sparse as sp

    return (u + sp.triu(u, 1).T).tocsr()


@pytest.mark.parametrize("spec", ["c5:5e3:50:0", "c1:0", "rqp:500:300:diagonal:0.02:5", "c2:1e4:5e3:0",
                                  "rqp:300:150:low_rank:0.05:3", "c3:2e3:100:0"])
@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_local_parts_hold_exactly_the_rank_rows(spec, nranks):
    """Storage shards: each rank's uploaded blocks reproduce its rows of A, A'
    and the full symmetric Q exactly (what the device builds from them), the
    local-nnz counts the device checks are right, and the windows cover every
    gathered column plus the rank's own rows."""
    p = instances.build(spec)
    plans = shard.plan(p, nranks)
    a = p.constraint_matrix.to_scipy().tocsr()
    at = a.T.tocsr()
    qf = _full_q(p)
    for r, me in enumerate(plans):
        part = shard.local_part(p, plans, r)
        blk_rows = me.ywin[1] - me.ywin[0]
        import scipy.sparse as sp

        blk = sp.csr_matrix((part.a_data, part.a_indices, part.a_indptr), shape=(blk_rows, p.n))
        # A rows [m0, m1) and A' rows [n0, n1) from the block
        assert (blk[me.m0 - me.ywin[0]:me.m1 - me.ywin[0]] != a[me.m0:me.m1]).nnz == 0
        assert me.a_local_nnz == a[me.m0:me.m1].nnz
        bt = blk.T.tocsr()[me.n0:me.n1]
        want = at[me.n0:me.n1]
        assert bt.nnz == want.nnz == me.at_local_nnz
        # the block's rows are global rows ywin[0] + local
        assert np.array_equal(np.sort(bt.indices + me.ywin[0]), np.sort(want.indices))
        c = [a[me.m0:me.m1].indices]
        if qf is not None:
            ub = sp.csr_matrix((part.q_data, part.q_indices, part.q_indptr), shape=(me.n1 - me.q_row0, p.n))
            full = sp.vstack([sp.csr_matrix((me.q_row0, p.n)), ub, sp.csr_matrix((p.n - me.n1, p.n))]).tocsr()
            rows = (full + sp.triu(full, 1).T).tocsr()[me.n0:me.n1]
            assert (rows != qf[me.n0:me.n1]).nnz == 0
            assert me.q_local_nnz == qf[me.n0:me.n1].nnz
            c.append(qf[me.n0:me.n1].indices)
        cols = np.concatenate(c)
        assert cols.size == 0 or (cols.min() >= me.xhalo[0] and cols.max() < me.xhalo[1])
        assert me.xwin[0] <= min(me.xhalo[0], me.n0) and me.xwin[1] >= max(me.xhalo[1], me.n1)
        ys = at[me.n0:me.n1].indices
        assert ys.size == 0 or (ys.min() >= me.yhalo[0] and ys.max() < me.yhalo[1])
        assert me.ywin[0] <= me.m0 and me.ywin[1] >= me.m1
        assert np.array_equal(part.cost, p.cost[me.n0:me.n1])
        assert np.array_equal(part.con_lo, p.con_bounds.lower[me.m0:me.m1])
        if p.quad.kind == "sparse_low_rank":  # columns [n0, n1) of R
            rr = p.quad.r.to_scipy().tocsc()[:, me.n0:me.n1].tocsr()
            if part.r_dense:
                assert np.array_equal(part.r_data.reshape(p.quad.r.rows, -1), rr.toarray())
            else:
                got = sp.csr_matrix((part.r_data, part.r_indices - me.n0, part.r_indptr), shape=rr.shape)
                assert (got != rr).nnz == 0


def test_banded_storage_shrinks_with_ranks():
    """C5-type (banded) windows are the rank's rows plus boundary strips, so a
    rank's stored rows and gather windows shrink ~1/P."""
    p = instances.build("c5:5e4:500:0")
    for P in (2, 4, 8):
        for me in shard.plan(p, P):
            assert (me.xwin[1] - me.xwin[0]) <= p.n / P + 2 * 1000 + 2
            assert (me.ywin[1] - me.ywin[0]) <= p.m / P + 2 * 600
            assert me.a_local_nnz + me.at_local_nnz + me.q_local_nnz <= 1.1 * (
                2 * p.constraint_matrix.nnz + 2 * p.quad.upper.nnz) / P


def _setup_worker(rank, world, port, q):
    """engine._setup_info over a gloo DistGroup with per-rank device structs
    faked: flags or-ed, first inverted index min-ed over the ranks that have
    one, maxima max-ed, R's row sums computed on the host for a low-rank Q."""
    import torch.distributed as dist

    from paper_2602_23967_b200 import _native as nat
    from paper_2602_23967_b200.engine import _setup_info

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = shard.DistGroup()

        class FakeDev:
            def setup_info(self):
                info = nat.SetupInfo()
                info.var_first_inverted = -1 if rank == 0 else 7
                info.con_first_inverted = 3 + rank
                info.q_nonfinite = rank
                info.con_scale, info.cost_inf = (2.0, 9.0) if rank == 0 else (3.5, 1.0)
                info.q_bound, info.r_one, info.diag_bound = 1.0 + rank, 4.0 - rank, 0.5 * rank
                info.r_inf_done = 0
                return info

        p = instances.build("rqp:300:150:low_rank:0.05:3")
        info = _setup_info(FakeDev(), p, g)
        q.put((rank, info.var_first_inverted, info.con_first_inverted, info.q_nonfinite, info.con_scale,
               info.cost_inf, info.q_bound, info.r_one, info.diag_bound, info.r_inf,
               float(p.quad.r.row_abs_sums().max(initial=0.0))))
    finally:
        dist.destroy_process_group()


def test_sharded_setup_info_combine_gloo_world2():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_setup_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    for r in res:
        _, vinv, cinv, qbad, cscale, cinf, qb, r1, db, rinf, rinf_host = r
        assert (vinv, cinv, qbad) == (7, 3, 1)
        assert (cscale, cinf, qb, r1, db) == (3.5, 9.0, 2.0, 4.0, 0.5)
        assert rinf == rinf_host
