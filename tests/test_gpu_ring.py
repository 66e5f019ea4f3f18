"""GPU: the banded ring path (spmv_ring_op) is bitwise the tile kernels.

The ring kernel keeps a window of the gathered vector in shared memory while
one CTA per SM walks a strip of row groups; each 256-row tile keeps its row ->
thread map, per-row summation order (the Cython order of `_core.pyx:62-80`) and
reduction tree, so a solve with the ring (AQP_RING unset) and one without it
(AQP_RING=0, spmv_op / spmv_sellp_op) must agree bit for bit: iterates, counts,
KKT and the norm estimate.
"""

import os

import numpy as np
import pytest

import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import generators
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem

pytestmark = pytest.mark.gpu


def _ring_mask(problem):
    return DeviceProblem(problem, DeviceContext.get(0)).info.ring_mask


KNOBS = ("AQP_RING", "AQP_RING_OFF", "AQP_RING_RT", "AQP_NO_SELL_ATTACH", "AQP_SELL")


def _solve(problem, ring, **kw):
    """ring: False (AQP_RING=0: tile kernels only), True (default policy) or
    a dict of ring knobs (AQP_RING_OFF op mask, AQP_RING_RT group size)."""
    env = {"AQP_RING": "0"} if ring is False else ({} if ring is True else dict(ring))
    saved = {k: os.environ.pop(k, None) for k in KNOBS}
    os.environ.update(env)
    try:
        return aq.solve(problem, aq.SolverParams(eps_tol=1e-8, **kw))
    finally:
        for k in KNOBS:
            os.environ.pop(k, None)
            if saved[k] is not None:
                os.environ[k] = saved[k]


def _same(r1, r2):
    assert r1.status == r2.status
    assert (r1.outer_iterations, r1.inner_iterations) == (r2.outer_iterations, r2.inner_iterations)
    assert np.array_equal(r1.x, r2.x) and np.array_equal(r1.y, r2.y)
    assert r1.report.kkt_max == r2.report.kkt_max


# default policy; every op on the ring (gradient and P1 too); the same with
# 512-row groups and two CTAs per SM
POLICIES = [True, {"AQP_RING_OFF": "0"}, {"AQP_RING_OFF": "0", "AQP_RING_RT": "512"}]


@pytest.mark.parametrize("n,w", [(400_000, 2000), (1_000_000, 5000)])
def test_ring_solve_bitwise_equals_tile_kernels(cuda, n, w):
    p = generators.banded_qp(n, n, half_width=w, seed=3)
    os.environ.pop("AQP_RING", None)
    assert _ring_mask(p) == 0b111  # A (SELL pairs), A' (SELL-P) and Q (plain SELL) windows planned
    want = _solve(p, False, iter_limit=40)
    for pol in POLICIES:
        _same(_solve(p, pol, iter_limit=40), want)


def test_ring_solve_to_optimal_matches(cuda):
    # a whole solve (restarts, certification, the norm estimate) through the ring
    p = generators.banded_qp(400_000, 400_000, half_width=300, seed=1)
    want = _solve(p, False)
    assert want.status == aq.SolveStatus.OPTIMAL
    for pol in POLICIES:
        _same(_solve(p, pol), want)


def test_ring_off_when_band_exceeds_ring(cuda):
    # A's +-9000 columns: a 1024-row group's window (~19k columns) exceeds
    # the 16384-entry ring -> A and A' run the tile kernels (Q's +-1000 band
    # still fits), same result
    p = generators.banded_qp(400_000, 400_000, half_width=9000, seed=2)
    os.environ.pop("AQP_RING", None)
    assert _ring_mask(p) == 0b100
    _same(_solve(p, True, iter_limit=10), _solve(p, False, iter_limit=10))


def test_ring_off_for_small_problems(cuda):
    # fewer than two groups per SM: no strip to walk
    p = generators.banded_qp(100_000, 100_000, half_width=500, seed=0)
    os.environ.pop("AQP_RING", None)
    assert _ring_mask(p) == 0


def test_unattached_sell_plans_deferred_at(cuda):
    # C5's A' (mean row 10 >= the staging threshold) defers its CSR plan to the
    # SELL-P attach; without the attach the solver plans it when created, and
    # the solve is bitwise the one planned at problem creation (no SELL at all).
    # (Not bitwise the SELL-P solve: A'-pass reductions -- the power
    # iteration's |A'w|^2 -- fold per plan item, and the CSR plan's STAGED
    # items are not the SELL-P plan's 256-row tiles.)
    p = generators.banded_qp(400_000, 400_000, half_width=2000, seed=4)
    want = _solve(p, {"AQP_SELL": "0"}, iter_limit=30)
    got = _solve(p, {"AQP_NO_SELL_ATTACH": "1"}, iter_limit=30)
    _same(got, want)
