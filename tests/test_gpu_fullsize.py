"""GPU: size-independent parity properties at BASELINE.json's full C5 size
(n = m = 5e7, 5e8 nonzeros in A, 2.5e8 in the full symmetric Q).

* the registry kernels (the drop-in C ABI) equal the oracle's C restatement of
  the Cython kernels BIT FOR BIT on the whole instance (row-sequential sums in
  the Cython order: A x, A'y through the explicit transpose, the symmetric Q x);
* the device setup scalars equal the host (numpy) values bitwise;
* two solves of the same instance are bitwise identical (deterministic
  reductions at full size);
* the banded ring path gives bitwise the tile kernels' solve.
"""

import numpy as np
import pytest

import oracle
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import certify, generators
from paper_2602_23967_b200 import kernels as kern
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem

pytestmark = pytest.mark.gpu

N, W = 50_000_000, 5000


@pytest.fixture(scope="module")
def c5():
    return generators.banded_qp(N, N, half_width=W, seed=0)


def test_registry_products_bitwise_oracle_full_c5(cuda, c5):
    a = c5.constraint_matrix
    rng = np.random.default_rng(1)
    x = rng.standard_normal(a.cols)
    y = rng.standard_normal(a.rows)
    assert np.array_equal(kern.csr_matvec(a.indptr, a.indices, a.data, x, a.rows),
                          oracle.csr_matvec(a.indptr, a.indices, a.data, x, a.rows))
    assert np.array_equal(kern.csr_matvec_t(a.indptr, a.indices, a.data, y, a.cols),
                          oracle.csr_matvec_t(a.indptr, a.indices, a.data, y, a.cols))
    q = c5.quad
    got = kern.sym_matvec(q.upper.indptr, q.upper.indices, q.upper.data, q.diag, x)
    want = oracle.sym_matvec(q.upper.indptr, q.upper.indices, q.upper.data, x)
    assert np.array_equal(got, want)


def test_setup_scalars_bitwise_full_c5(cuda, c5):
    info = DeviceProblem(c5, DeviceContext.get(0)).setup_info()
    assert 1.0 + info.q_bound == certify.default_gamma_sys(c5)
    assert info.con_scale == certify.finite_bound_scale(c5.con_bounds)
    assert info.cost_inf == certify.linf(c5.cost)
    assert info.diag_bound == c5.quad.diag_bound()


def test_solve_deterministic_full_c5(cuda, c5):
    prm = aq.SolverParams(eps_tol=1e-8, iter_limit=3)
    r1, r2 = aq.solve(c5, prm), aq.solve(c5, prm)
    assert (r1.outer_iterations, r1.inner_iterations) == (r2.outer_iterations, r2.inner_iterations)
    assert np.array_equal(r1.x, r2.x) and np.array_equal(r1.y, r2.y)
    assert r1.report.kkt_max == r2.report.kkt_max


def test_ring_path_bitwise_tile_kernels_full_c5(cuda, c5):
    # the banded ring path (spmv_ring_op: P2 and the power iteration by
    # default, every op with AQP_RING_OFF=0) against the tile kernels only
    # (AQP_RING=0), at the full size: iterates, counts and KKT bit for bit
    import os

    prm = aq.SolverParams(eps_tol=1e-8, iter_limit=3)
    runs = []
    for env in ({"AQP_RING": "0"}, {}, {"AQP_RING_OFF": "0"}):
        saved = {k: os.environ.pop(k, None) for k in ("AQP_RING", "AQP_RING_OFF")}
        os.environ.update(env)
        try:
            runs.append(aq.solve(c5, prm))
        finally:
            for k, v in saved.items():
                os.environ.pop(k, None)
                if v is not None:
                    os.environ[k] = v
    want = runs[0]
    for r in runs[1:]:
        assert (r.outer_iterations, r.inner_iterations) == (want.outer_iterations, want.inner_iterations)
        assert np.array_equal(r.x, want.x) and np.array_equal(r.y, want.y)
        assert r.report.kkt_max == want.report.kkt_max
