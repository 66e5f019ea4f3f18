"""ctypes binding of libaqp.so (include/aqp.h).

The library is REQUIRED: importing this module on a machine without the
built library or without a CUDA device raises ``DeviceError`` -- there is no
host fallback for any product call.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, InvalidProblem, TooLarge, ZeroMatrix

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaqp.so")

AQP_OK, AQP_EINVAL, AQP_ECUDA, AQP_ENOMEM, AQP_ERANGE, AQP_EZERO, AQP_ESTATE = 0, -1, -2, -3, -4, -5, -6
QUAD_DIAGONAL, QUAD_SPARSE, QUAD_SPARSE_LOW_RANK = 0, 1, 2

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


ABI_VERSION = 3


class ShardDesc(C.Structure):
    """aqp_shard_desc: this rank's rows, uploaded blocks and every rank's gather windows."""

    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("n0", C.c_int64), ("n1", C.c_int64),
                ("m0", C.c_int64), ("m1", C.c_int64), ("a_row0", C.c_int64), ("a_rows", C.c_int64),
                ("q_row0", C.c_int64), ("a_local_nnz", C.c_int64), ("at_local_nnz", C.c_int64),
                ("q_local_nnz", C.c_int64), ("xw", C.c_int64 * 16), ("yw", C.c_int64 * 16),
                ("nl_cap", C.c_int64), ("ml_cap", C.c_int64)]


class ProblemDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("m", C.c_int64),
        ("a_indptr", C.c_void_p), ("a_indices", C.c_void_p), ("a_data", C.c_void_p), ("a_nnz", C.c_int64),
        ("quad_kind", C.c_int32),
        ("q_values", C.c_void_p),
        ("q_indptr", C.c_void_p), ("q_indices", C.c_void_p), ("q_data", C.c_void_p), ("q_nnz", C.c_int64),
        ("q_diag", C.c_void_p),
        ("r_rows", C.c_int64),
        ("r_indptr", C.c_void_p), ("r_indices", C.c_void_p), ("r_data", C.c_void_p), ("r_nnz", C.c_int64),
        ("r_dense", C.c_int32), ("pad0_", C.c_int32),
        ("cost", C.c_void_p), ("var_lo", C.c_void_p), ("var_hi", C.c_void_p),
        ("con_lo", C.c_void_p), ("con_hi", C.c_void_p),
        ("shard", C.c_void_p),
    ]


class ProblemInfo(C.Structure):
    _fields_ = [
        ("a_nnz", C.c_int64), ("at_nnz", C.c_int64), ("q_full_nnz", C.c_int64), ("r_rows", C.c_int64),
        ("a_items", C.c_int64), ("at_items", C.c_int64), ("q_items", C.c_int64),
        ("quad_kind", C.c_int32), ("r_dense", C.c_int32),
        ("persistent_bytes", C.c_size_t),
        ("ring_mask", C.c_int32),
    ]


class SetupInfo(C.Structure):
    _fields_ = [
        ("var_nan", C.c_int32), ("var_wrong_inf", C.c_int32), ("con_nan", C.c_int32), ("con_wrong_inf", C.c_int32),
        ("var_first_inverted", C.c_int64), ("con_first_inverted", C.c_int64),
        ("cost_nonfinite", C.c_int32), ("a_nonfinite", C.c_int32), ("q_nonfinite", C.c_int32),
        ("r_inf_done", C.c_int32),
        ("con_scale", C.c_double), ("cost_inf", C.c_double), ("q_bound", C.c_double), ("r_one", C.c_double),
        ("r_inf", C.c_double), ("diag_bound", C.c_double),
    ]


class SolverParamsC(C.Structure):
    _fields_ = [
        ("eps_tol", C.c_double), ("eps_inf", C.c_double), ("gamma_sys", C.c_double),
        ("tol_scale", C.c_double), ("tol_floor", C.c_double), ("diag_bound", C.c_double),
        ("adaptive", C.c_int32), ("max_inner", C.c_int32), ("halpern", C.c_int32), ("pad_", C.c_int32),
    ]


class Scalars(C.Structure):
    _fields_ = [
        ("eta", C.c_double), ("omega", C.c_double), ("theta", C.c_double), ("inner_tol", C.c_double),
        ("k", C.c_int64), ("probing", C.c_int32), ("halted", C.c_int32),
        ("iters_done", C.c_int64), ("inner_sum", C.c_int64), ("block_len", C.c_int64),
        ("have_avg_prev", C.c_int32), ("pad_", C.c_int32),
    ]


class CheckResult(C.Structure):
    _fields_ = [
        ("primal_viol", C.c_double), ("dual_viol", C.c_double), ("qx_inf", C.c_double), ("aty_inf", C.c_double),
        ("pr_pos", C.c_double), ("pr_neg", C.c_double), ("py_pos", C.c_double), ("py_neg", C.c_double),
        ("xqx", C.c_double), ("cx", C.c_double), ("pid_dx2", C.c_double), ("pid_dy2", C.c_double),
        ("pr_bad", C.c_int32), ("py_bad", C.c_int32), ("have_avg_prev", C.c_int32), ("pad_", C.c_int32),
        ("yr_norm", C.c_double * 2), ("yr_viol", C.c_double * 2), ("yr_aty_inf", C.c_double * 2),
        ("yr_var_pos", C.c_double * 2), ("yr_var_neg", C.c_double * 2),
        ("yr_con_pos", C.c_double * 2), ("yr_con_neg", C.c_double * 2),
        ("yr_var_bad", C.c_int32 * 2), ("yr_con_bad", C.c_int32 * 2),
        ("xr_norm", C.c_double * 2), ("xr_improvement", C.c_double * 2), ("xr_viol_x", C.c_double * 2),
        ("xr_viol_s", C.c_double * 2), ("xr_qd_inf", C.c_double * 2),
    ]


# exported symbol -> (restype, argtypes); mirrors include/aqp.h one to one
_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
SIGNATURES = {
    "aqp_abi_version": (C.c_int, []),
    "aqp_last_error": (C.c_char_p, []),
    "aqp_csr_matvec": (C.c_int, [_P, _P, _P, _P, _I64, _I64, _P]),
    "aqp_csr_matvec_t": (C.c_int, [_P, _P, _P, _P, _I64, _I64, _P]),
    "aqp_sym_matvec": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P]),
    "aqp_clamp": (C.c_int, [_P, _P, _P, _I64, _P]),
    "aqp_cone_project": (C.c_int, [_P, _P, _I64, _P]),
    "aqp_diag_prox_step": (C.c_int, [_P, _P, _P, _D, _P, _P, _I64, _P]),
    "aqp_natural_res_sq": (C.c_int, [_P, _P, _P, _P, _I64, _P]),
    "aqp_dual_step": (C.c_int, [_P, _P, _D, _P, _P, _I64, _P]),
    "aqp_lincomb3": (C.c_int, [_D, _P, _D, _P, _D, _P, _I64, _P]),
    "aqp_axpby": (C.c_int, [_D, _P, _D, _P, _I64, _P]),
    "aqp_support_p": (C.c_int, [_P, _P, _P, _I64, _P]),
    "aqp_ctx_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "aqp_ctx_destroy": (C.c_int, [_P]),
    "aqp_problem_sizes": (C.c_int, [C.POINTER(ProblemDesc), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "aqp_problem_create": (C.c_int, [_P, C.POINTER(ProblemDesc), _P, _P, _P, _P, C.c_size_t, _P, C.c_size_t,
                                     C.POINTER(_P)]),
    "aqp_problem_get_info": (C.c_int, [_P, C.POINTER(ProblemInfo)]),
    "aqp_problem_destroy": (C.c_int, [_P]),
    "aqp_problem_setup_info": (C.c_int, [_P, C.POINTER(SetupInfo)]),
    "aqp_problem_sell_bytes": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "aqp_problem_attach_sell": (C.c_int, [_P, _P, C.c_size_t]),
    "aqp_h2d": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "aqp_d2h": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "aqp_solver_sizes": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "aqp_solver_create": (C.c_int, [_P, C.POINTER(SolverParamsC), _P, C.c_size_t, C.POINTER(_P)]),
    "aqp_solver_destroy": (C.c_int, [_P]),
    "aqp_solver_init": (C.c_int, [_P, C.POINTER(Scalars)]),
    "aqp_solver_set_scalars": (C.c_int, [_P, C.POINTER(Scalars)]),
    "aqp_solver_get_scalars": (C.c_int, [_P, C.POINTER(Scalars)]),
    "aqp_solver_run": (C.c_int, [_P, _I64]),
    "aqp_solver_check": (C.c_int, [_P, C.c_int, C.POINTER(CheckResult)]),
    "aqp_solver_mark_cert": (C.c_int, [_P]),
    "aqp_solver_restart": (C.c_int, [_P]),
    "aqp_solver_rollback": (C.c_int, [_P]),
    "aqp_solver_reset_window": (C.c_int, [_P]),
    "aqp_solver_read": (C.c_int, [_P, C.c_int, _P, _I64]),
    "aqp_solver_counters": (C.c_int, [_P, c_int64_p]),
    "aqp_solver_estimate_norm": (C.c_int, [_P, _P, C.c_int, c_double_p, C.POINTER(C.c_int)]),
    "aqp_solver_time_kernel": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_size_t, c_double_p]),
    "aqp_solver_trace": (C.c_int, [_P, _P, _I64, c_int64_p]),
    # scaled solves (opt-in Ruiz / Pock-Chambolle)
    "aqp_problem_scale": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P, C.c_size_t]),
    "aqp_solver_import_scaled": (C.c_int, [_P, _P, _P, _P]),
    # row shards (multi-GPU)
    "aqp_solver_exchange_region": (C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_size_t)]),
    "aqp_solver_connect": (C.c_int, [_P, C.POINTER(_P), C.c_int]),
    "aqp_solver_set_halos": (C.c_int, [_P, c_int64_p, c_int64_p, C.c_int]),
    "aqp_ipc_get_handle": (C.c_int, [_P, _P, C.POINTER(C.c_size_t)]),
    "aqp_ipc_open": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "aqp_ipc_close": (C.c_int, [_P, C.c_size_t]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libaqp.so and bind every exported symbol (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"libaqp.so not built at {path}; run `python -m paper_2602_23967_b200.build`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.aqp_abi_version() != ABI_VERSION:
        raise DeviceError("libaqp ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map an AQP_E* code to the package's error classes."""
    if rc == AQP_OK:
        return
    msg = (_lib.aqp_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == AQP_EINVAL:
        raise InvalidProblem(text)
    if rc == AQP_ERANGE:
        raise TooLarge(text)
    if rc == AQP_EZERO:
        raise ZeroMatrix(text)
    raise DeviceError(f"[{rc}] {text}")


def ptr(arr) -> int:
    """Address of a contiguous numpy array or torch tensor."""
    if hasattr(arr, "data_ptr"):
        return arr.data_ptr()
    return arr.ctypes.data
