"""The CPU oracle is pinned to the real reference before anything is checked
against it: its kernels reproduce the reference's Cython kernels bit for bit
(golden vectors recorded from oracle/_ref by oracle/gen_golden_kernels.py) and
its solve loop reproduces the reference's golden runs exactly (recorded by
oracle/run_reference.py)."""

import os

import numpy as np
import pytest

import instances
import oracle
from conftest import GOLDEN, golden
from paper_2602_23967_b200 import SolverParams

K = np.load(os.path.join(GOLDEN, "kernels.npz"))


@pytest.mark.parametrize("t", range(5))
def test_oracle_csr_kernels_bitwise(t):
    ip, ix, dv = K[f"mv{t}_indptr"], K[f"mv{t}_indices"], K[f"mv{t}_data"]
    rows, cols = len(ip) - 1, len(K[f"mv{t}_x"])
    assert np.array_equal(oracle.csr_matvec(ip, ix, dv, K[f"mv{t}_x"], rows), K[f"mv{t}_ax"])
    assert np.array_equal(oracle.csr_matvec_t(ip, ix, dv, K[f"mv{t}_y"], cols), K[f"mv{t}_aty"])


@pytest.mark.parametrize("t", range(4))
def test_oracle_sym_kernel_bitwise(t):
    out = oracle.sym_matvec(K[f"sym{t}_indptr"], K[f"sym{t}_indices"], K[f"sym{t}_data"], K[f"sym{t}_x"])
    assert np.array_equal(out, K[f"sym{t}_out"])


def test_oracle_vector_kernels_bitwise():
    x, g, q, lin, lo, hi = (K[k] for k in ("v_x", "v_g", "v_q", "v_lin", "v_lo", "v_hi"))
    assert np.array_equal(oracle.clamp(x, lo, hi), K["k_clamp"])
    assert np.array_equal(oracle.cone_project(x, K["v_codes"]), K["k_cone"])
    assert np.array_equal(oracle.diag_prox_step(x, q, lin, 0.37, lo, hi), K["k_prox"])
    assert oracle.natural_res_sq(x, g, lo, hi) == K["k_natres"][0]
    assert np.array_equal(oracle.dual_step(x, g, 1.7, lo, hi), K["k_dual"])
    assert np.array_equal(oracle.lincomb3(0.3, x, 0.6, g, -0.25, lin), K["k_lin3"])
    assert np.array_equal(oracle.axpby(2.0, x, -1.0, g), K["k_axpby"])
    z = x * (np.isfinite(lo) & np.isfinite(hi))
    assert oracle.support(z, lo, hi) == K["k_support"][0]


GOLDEN_RUNS = [
    ("c1:0", "ref_c1_s0.json"),
    ("c4ur:1e3:1", "ref_c4ur_1e3_1.json"),
    ("c4ir:1e3:1", "ref_c4ir_1e3_1.json"),
    ("rqp:300:150:sparse:0.05:7", "ref_rqp_300_150_sparse_0.05_7.json"),
    ("rqp:300:150:low_rank:0.05:3", "ref_rqp_300_150_low_rank_0.05_3.json"),
    ("rqp:500:300:diagonal:0.02:5", "ref_rqp_500_300_diagonal_0.02_5.json"),
]


@pytest.mark.parametrize("spec,fname", GOLDEN_RUNS)
def test_oracle_reproduces_reference_runs(spec, fname):
    g = golden(fname)
    r = oracle.solve(instances.build(spec), SolverParams(eps_tol=g["eps_tol"]))
    assert r["status"] == g["status"]
    assert (r["outer"], r["inner"], r["restarts"]) == (g["outer"], g["inner"], g["restarts"])
    assert r["report"]["primal_objective"] == g["objective"]
    assert r["report"]["kkt"] == g["kkt"]


def test_norm_memo_is_the_reference_value():
    """bench.py's reference arm serves estimate_norm from oracle/norm_memo.py's
    recordings; a recording must be bitwise what the unmodified reference
    function returns on the same matrix, and an unrecorded matrix must fall
    through to the real function."""
    import norm_memo
    import refbridge

    aq = refbridge.load_reference()
    if aq is None:
        pytest.skip("reference not built (oracle/build_ref.sh)")
    import anchorqp.engine as eng
    import anchorqp.linalg as L

    prob = refbridge.to_reference(instances.build("c5:5e4:500:0"), aq)
    live = L.estimate_norm(prob.constraint_matrix, 100, 0)
    rec = norm_memo._load()[norm_memo.fingerprint(prob.constraint_matrix)]
    assert float.fromhex(rec["value_hex"]) == live
    saved = eng.estimate_norm
    try:
        f = norm_memo.patch(aq)
        assert eng.estimate_norm is f
        assert f(prob.constraint_matrix, 100, 0) == live  # recorded, bitwise
        other = refbridge.to_reference(instances.build("c5:2e3:50:1"), aq).constraint_matrix
        assert f(other, 20, 0) == L.estimate_norm(other, 20, 0)  # not recorded: the real function
    finally:
        eng.estimate_norm = saved
