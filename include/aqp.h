/*
 * aqp.h -- C ABI of libaqp, the B200 (sm_100a) implementation of the PDHCG-II
 * solve loop of the reference package `anchorqp`.
 *
 * Two boundaries are exported, both plain C (no torch / numpy types):
 *
 * 1. The kernel-registry boundary (section "registry"): one entry point per
 *    name in the reference registry, anchorqp/_kernels/__init__.py:16-27, with
 *    the argument meaning of the Cython module anchorqp/_kernels/_core.pyx.
 *    They take HOST pointers (like the Cython kernels take numpy buffers),
 *    copy to HBM, run the sm_100a kernel and copy the result back, so a
 *    ctypes stub can register them as a drop-in backend.
 *
 * 2. The solver boundary (sections "context" .. "solver"): the device-resident
 *    state machine that the Python `solve()` (anchorqp/engine.py:339-498
 *    restated) drives.  Device memory is supplied by the caller (PyTorch
 *    tensors) as workspaces whose sizes the library reports.
 *
 * Every function returns 0 on success or a negative AQP_E* code; the message
 * of the last failure on the calling thread is aqp_last_error().
 */
#ifndef AQP_H_
#define AQP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AQP_ABI_VERSION 3

enum {
  AQP_OK = 0,
  AQP_EINVAL = -1,   /* bad argument / malformed data (maps to InvalidProblem) */
  AQP_ECUDA = -2,    /* CUDA runtime error (DeviceError)                      */
  AQP_ENOMEM = -3,   /* workspace too small / device OOM                        */
  AQP_ERANGE = -4,   /* size exceeds int32 device indexing (TooLarge)          */
  AQP_EZERO = -5,    /* all-zero matrix where a norm is needed (ZeroMatrix)     */
  AQP_ESTATE = -6    /* call out of order                                       */
};

/* cone codes, reference anchorqp/_kernels/__init__.py:14 */
enum { AQP_ZERO = 0, AQP_NONNEG = 1, AQP_NONPOS = 2, AQP_FREE = 3 };

/* quadratic operator kinds, reference anchorqp/linalg.py:147,177,230 */
enum { AQP_QUAD_DIAGONAL = 0, AQP_QUAD_SPARSE = 1, AQP_QUAD_SPARSE_LOW_RANK = 2 };

int aqp_abi_version(void);
const char *aqp_last_error(void);

/* ------------------------------------------------------------------------ */
/* registry: drop-in replacements of anchorqp/_kernels/_core.pyx            */
/* Host pointers in, host pointer out (caller-allocated, length as noted).  */
/* Executed on the library's own stream on the current device.              */
/* ------------------------------------------------------------------------ */

/* _core.pyx:29-42  out[nrows] = A x  (row-sequential sum, Cython order)     */
int aqp_csr_matvec(const int64_t *indptr, const int64_t *indices, const double *data,
                   const double *x, int64_t nrows, int64_t ncols, double *out);
/* _core.pyx:45-59  out[ncols] = A' x  (explicit transpose, ascending rows)  */
int aqp_csr_matvec_t(const int64_t *indptr, const int64_t *indices, const double *data,
                     const double *x, int64_t nrows, int64_t ncols, double *out);
/* _core.pyx:62-80  out[n] = S x, S symmetric given by its upper triangle     */
int aqp_sym_matvec(const int64_t *indptr, const int64_t *indices, const double *data,
                   const double *diag, const double *x, int64_t n, double *out);
/* _core.pyx:83-92 */
int aqp_clamp(const double *x, const double *lo, const double *hi, int64_t n, double *out);
/* _core.pyx:95-115 */
int aqp_cone_project(const double *z, const int8_t *codes, int64_t n, double *out);
/* _core.pyx:118-128 */
int aqp_diag_prox_step(const double *xk, const double *q, const double *linear, double tau,
                       const double *lo, const double *hi, int64_t n, double *out);
/* _core.pyx:131-142  (returns the sum through *out) */
int aqp_natural_res_sq(const double *x, const double *g, const double *lo, const double *hi,
                       int64_t n, double *out);
/* _core.pyx:145-157 */
int aqp_dual_step(const double *y, const double *ax, double sigma, const double *lo,
                  const double *hi, int64_t m, double *out);
/* _core.pyx:160-170 */
int aqp_lincomb3(double a, const double *x, double b, const double *y, double c,
                 const double *z, int64_t n, double *out);
/* _core.pyx:173-182 */
int aqp_axpby(double a, const double *x, double b, const double *y, int64_t n, double *out);
/* model.py:57-71 support function of a box (0*inf = 0, +inf on a bad side) */
int aqp_support_p(const double *z, const double *lo, const double *hi, int64_t n, double *out);

/* ------------------------------------------------------------------------ */
/* context                                                                   */
/* ------------------------------------------------------------------------ */
typedef struct aqp_ctx aqp_ctx;
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) */
int aqp_ctx_create(int device, void *stream, aqp_ctx **out);
int aqp_ctx_destroy(aqp_ctx *ctx);

/* ------------------------------------------------------------------------ */
/* problem: device copy of QpProblem (reference model.py:124-165)            */
/* ------------------------------------------------------------------------ */
/* Storage shard of a row-partitioned problem (the
 * reference has no multi-GPU path -- its only parallelism is a process pool
 * over instances, anchorqp/bench.py:89-98).  Rank `rank` of `nranks` (<= 8)
 * owns rows [n0,n1) of A' and of the full symmetric Q (x side) and rows
 * [m0,m1) of A (y side), and stores ONLY those: with a shard descriptor the
 * aqp_problem_desc arrays are this rank's blocks (see aqp_problem_desc).
 * Gathered vectors live in per-rank windows [xw[2r], xw[2r+1]) /
 * [yw[2r], yw[2r+1]) that cover the rank's own rows and every column its
 * rows gather; column indices stay global.  All ranks pass identical xw /
 * yw tables (they size the peer-visible exchange region identically). */
typedef struct {
  int32_t rank, nranks;
  int64_t n0, n1, m0, m1;   /* owned rows */
  int64_t a_row0, a_rows;   /* the uploaded A block: rows [a_row0, a_row0 + a_rows) of A, covering
                               [m0,m1) and every row with a nonzero in columns [n0,n1) */
  int64_t q_row0;           /* the uploaded P block: upper-triangle rows [q_row0, n1), covering every
                               row with an upper entry in columns [n0,n1) */
  int64_t a_local_nnz;      /* nonzeros of A rows [m0,m1) */
  int64_t at_local_nnz;     /* nonzeros of the A block in columns [n0,n1) (= nnz of A' rows [n0,n1)) */
  int64_t q_local_nnz;      /* nonzeros of full symmetric Q rows [n0,n1) (diagonal included) */
  int64_t xw[16], yw[16];   /* gather windows of every rank: [lo, hi) pairs, rank-major */
  int64_t nl_cap, ml_cap;   /* max over ranks of n1-n0 and m1-m0 */
} aqp_shard_desc;

/* All array pointers are DEVICE pointers to the reference layouts
 * (CSR int64 indptr/indices, float64 values, float64 vectors), already in
 * HBM.  They are read during aqp_problem_create only.
 *
 * With `shard` set (a row shard, see aqp_shard_desc) the arrays are this
 * rank's blocks, indices global: a_* = the A block (a_rows rows), q_* = the
 * upper-triangle P block (rows [q_row0, n1)), q_values / q_diag / cost /
 * var_lo / var_hi = entries [n0,n1), con_lo / con_hi = entries [m0,m1),
 * r_* = columns [n0,n1) of R (dense: r_rows x (n1-n0) row-major; CSR:
 * r_rows rows with global column indices). */
typedef struct {
  int64_t n, m;
  /* A: m x n CSR (linalg.py:28-112) */
  const int64_t *a_indptr;
  const int64_t *a_indices;
  const double *a_data;
  int64_t a_nnz;
  /* Q */
  int32_t quad_kind;
  const double *q_values; /* DIAGONAL: n entries */
  const int64_t *q_indptr; /* SPARSE / LOW_RANK: upper-triangle CSR of P */
  const int64_t *q_indices;
  const double *q_data;
  int64_t q_nnz;
  const double *q_diag;    /* diagonal of P (n) */
  /* LOW_RANK: R is r_rows x n CSR */
  int64_t r_rows;
  const int64_t *r_indptr;
  const int64_t *r_indices;
  const double *r_data;
  int64_t r_nnz;
  /* LOW_RANK: every row of R is full (indptr = i*n, indices = 0..n-1), so
   * r_data IS R dense row-major (r_rows x n); r_indices is not read.  The
   * factor-model case (linalg.py:230-266 with R = F'): held dense on the
   * device, R x and R'v become streaming passes (16 B per entry per apply
   * instead of 24 B of CSR for R plus R'). */
  int32_t r_dense;
  int32_t pad0_;
  /* vectors */
  const double *cost;   /* n */
  const double *var_lo; /* n */
  const double *var_hi; /* n */
  const double *con_lo; /* m */
  const double *con_hi; /* m */
  const aqp_shard_desc *shard; /* NULL: the whole problem on this device */
} aqp_problem_desc;

typedef struct {
  int64_t a_nnz, at_nnz, q_full_nnz, r_rows;
  int64_t a_items, at_items, q_items;   /* SpMV work items (blocks) per pass */
  int32_t quad_kind, r_dense;
  size_t persistent_bytes;
  int32_t ring_mask;  /* bit 0 / 1 / 2: A / A' / Q passes may use the banded
                         ring kernel (set by aqp_problem_attach_sell) */
} aqp_problem_info;

typedef struct aqp_problem aqp_problem;
/* Bytes of the persistent workspace (kept for the problem's lifetime) and of
 * the transient scratch (needed only inside aqp_problem_create). */
int aqp_problem_sizes(const aqp_problem_desc *desc, size_t *persistent_bytes, size_t *scratch_bytes);
/* host_a_indptr / host_q_indptr / host_r_indptr: HOST copies of the indptr
 * arrays (used to plan the SpMV work partition; may be NULL for absent parts;
 * for a shard: of the uploaded blocks). */
int aqp_problem_create(aqp_ctx *ctx, const aqp_problem_desc *desc,
                       const int64_t *host_a_indptr, const int64_t *host_q_indptr,
                       const int64_t *host_r_indptr,
                       void *persistent, size_t persistent_bytes,
                       void *scratch, size_t scratch_bytes, aqp_problem **out);
int aqp_problem_get_info(const aqp_problem *p, aqp_problem_info *out);
/* Optional coalesced SELL-32 copies of the uniform short-row matrices (A,
 * A', Q, R, R' whose every row fits one thread and whose 32-row slices pad
 * <= 1/8): the SpMV passes then load a warp's k-th nonzeros contiguously
 * (C5: A x 2.57 -> 2.07 ms, Q x 1.25 -> 1.17 ms).  The layout is planned in
 * aqp_problem_create; the caller supplies device memory of
 * aqp_problem_sell_bytes (0: nothing to attach) and attaches it before
 * creating solvers.  The buffer must outlive the problem. */
int aqp_problem_sell_bytes(const aqp_problem *p, size_t *bytes);
int aqp_problem_attach_sell(aqp_problem *p, void *buf, size_t bytes);

/* Device-side Ruiz (ruiz_iters rounds of inf-norm equilibration of
 * K = [[Q, A'], [A, 0]]) and optional Pock-Chambolle (alpha = 1, l1) scaling,
 * applied IN PLACE to the device problem (A, A', Q, R, c, bounds).  D (n) and
 * E (m) receive the scalings (device buffers); the solve of the scaled problem
 * maps back by x = D x~, y = E y~.  Opt-in (not in the reference: the default
 * solve never scales).  scratch: >= (2 n + m) doubles of device memory. */
int aqp_problem_scale(aqp_problem *p, int ruiz_iters, int pock_chambolle, double *D, double *E, void *scratch,
                      size_t scratch_bytes);
int aqp_problem_destroy(aqp_problem *p);

/* Validation flags and setup scalars of a created problem, computed on the
 * device (replaces the host passes of anchorqp's solve entry):
 *   model.py:168-206   validate(): the host raises the FIRST violation in the
 *                      reference's order (var bounds, con bounds, cost, A, Q)
 *   certify.py:54-60   finite_bound_scale(con_bounds) -> con_scale; |c|_inf
 *   linalg.py:218-220  SparseQuad.inf_norm_bound (bitwise: sequential row /
 *                      column sums in numpy.bincount's order) -> q_bound
 *                      (DIAGONAL: max(values))
 *   linalg.py:260-263  low rank: r_one = max col abs sum of R, r_inf = max row
 *                      abs sum (r_inf_done = 0 for a row shard: R's rows span
 *                      every rank's columns, the host computes it)
 *   linalg.py:167-168,215-216,252-258  diag_bound
 * Indices are global; a row shard reports its own rows / columns (maxima,
 * flags and first indices combine across ranks by max / or / min). */
typedef struct {
  int32_t var_nan, var_wrong_inf, con_nan, con_wrong_inf;
  int64_t var_first_inverted, con_first_inverted;  /* -1: none */
  int32_t cost_nonfinite, a_nonfinite, q_nonfinite, r_inf_done;
  double con_scale, cost_inf, q_bound, r_one, r_inf, diag_bound;
} aqp_setup_info;
int aqp_problem_setup_info(aqp_problem *p, aqp_setup_info *out);

/* Bulk synchronous copies between host memory (pageable, e.g. numpy) and
 * device memory of ctx's device, staged through a process-wide pool of
 * pinned buffers by 8 host threads (~45 GB/s H2D on the B200 box vs ~10 GB/s
 * pageable).  aqp_d2h first synchronises ctx's stream (the source is
 * produced there). */
int aqp_h2d(aqp_ctx *ctx, void *dev_dst, const void *host_src, size_t bytes);
int aqp_d2h(aqp_ctx *ctx, void *host_dst, const void *dev_src, size_t bytes);



/* ------------------------------------------------------------------------ */
/* solver: device-resident iteration state (engine.py:125-155 + solve locals) */
/* ------------------------------------------------------------------------ */
typedef struct {
  double eps_tol, eps_inf;
  double gamma_sys;
  double tol_scale, tol_floor;
  double diag_bound;       /* QuadOperator.diag_bound(), inner.py:102 */
  int32_t adaptive;
  int32_t max_inner;
  int32_t halpern;
  int32_t pad_;
} aqp_solver_params;

/* scalar state shared between host logic and device kernels */
typedef struct {
  double eta, omega, theta;
  double inner_tol;        /* InnerTolerance.current (inner.py:28-38) */
  int64_t k;               /* Halpern counter k_inner_halpern */
  int32_t probing;         /* window runs plain PDHG steps (engine.py:396-403) */
  int32_t halted;          /* a step produced a non-finite move (engine.py:407) */
  int64_t iters_done;      /* outer iterations completed in the last window */
  int64_t inner_sum;       /* BB iterations accumulated over the last window */
  int64_t block_len;       /* window-sum length (engine.py:391,428) */
  int32_t have_avg_prev;   /* x_avg_prev/y_avg_prev exist (engine.py:450) */
  int32_t pad_;
} aqp_scalars;

/* Raw reductions of one certification point.  The host restates the
 * residual / certificate formulas of certify.py:63-164 on these numbers, so
 * the comparisons (and Python's max/min NaN behaviour) are the reference's. */
typedef struct {
  /* residuals(x_eval, y), certify.py:63-95 */
  double primal_viol;           /* |Ax - proj_S(Ax)|_inf                    */
  double dual_viol;             /* |r - proj_R(r)|_inf, r = Qx + c + A'y     */
  double qx_inf, aty_inf;       /* |Qx|_inf, |A'y|_inf                       */
  double pr_pos, pr_neg;        /* support_p(-proj_R r; l_v, u_v) = pos + neg */
  double py_pos, py_neg;        /* support_p(proj_Y y; l_c, u_c)             */
  double xqx, cx;               /* x'Qx, c'x                                 */
  double pid_dx2, pid_dy2;      /* |x - x_rs|^2, |y - y_rs|^2 (engine.py:267) */
  int32_t pr_bad, py_bad;       /* support value is +inf                     */
  int32_t have_avg_prev, pad_;
  /* y-ray candidates j = 0 (window-average difference), 1 (since last check):
   * certify.py:109-133 on proj_Y(dy)/|proj_Y(dy)|_inf */
  double yr_norm[2], yr_viol[2], yr_aty_inf[2];
  double yr_var_pos[2], yr_var_neg[2], yr_con_pos[2], yr_con_neg[2];
  int32_t yr_var_bad[2], yr_con_bad[2];
  /* x-ray candidates: certify.py:136-164 on d = dx/|dx|_inf (viol_s / qd_inf
   * are only evaluated when improvement < -eps_tol) */
  double xr_norm[2], xr_improvement[2], xr_viol_x[2], xr_viol_s[2], xr_qd_inf[2];
} aqp_check_result;

typedef struct aqp_solver aqp_solver;
int aqp_solver_sizes(const aqp_problem *p, size_t *workspace_bytes);
int aqp_solver_create(aqp_problem *p, const aqp_solver_params *params, void *workspace,
                      size_t workspace_bytes, aqp_solver **out);
int aqp_solver_destroy(aqp_solver *s);
/* Scaled solves: dst (a solver of the ORIGINAL problem) <- the current
 * iterate, anchor and window sums of src (a solver of the aqp_problem_scale'd
 * problem) mapped back by x = D x~, y = E y~; then aqp_solver_check(dst, ...)
 * certifies on the original problem.  Both solvers must share a stream. */
int aqp_solver_import_scaled(aqp_solver *dst, aqp_solver *src, const double *D, const double *E);
/* Row shards: the front of the solver workspace (every gathered vector and
 * the exchange mailbox) is written by the peers; its layout is identical on
 * every rank (buffers are sized by the shard descriptor's max-over-ranks
 * capacities).  After every rank's aqp_solver_create has returned (host
 * barrier), pass each rank's mapping of its peers' workspace bases
 * (peer_bases[rank] = this workspace; CUDA IPC mappings across processes,
 * plain pointers for ranks sharing a device).  Builds the window graph.
 * From then on every aqp_solver_* call is collective: all ranks make the
 * same calls in the same order. */
int aqp_solver_exchange_region(aqp_solver *s, void **base, size_t *bytes);
int aqp_solver_connect(aqp_solver *s, void *const *peer_bases, int nranks);
/* Before aqp_solver_connect: the gather halos of every rank.  Rank k gathers
 * x only in [x_lohi[2k], x_lohi[2k+1]) (columns of its rows of A and Q) and
 * y only in [y_lohi[2k], y_lohi[2k+1]) (columns of its rows of A');
 * producers store to peer k only entries inside k's range, which must lie
 * inside k's gather window.  Default: the windows. */
int aqp_solver_set_halos(aqp_solver *s, const int64_t *x_lohi, const int64_t *y_lohi, int nranks);
/* x0 = clamp(0), y0 = 0, all round/anchor buffers <- (x0, y0) (engine.py:174-204) */
int aqp_solver_init(aqp_solver *s, const aqp_scalars *sc);
int aqp_solver_set_scalars(aqp_solver *s, const aqp_scalars *sc);
int aqp_solver_get_scalars(aqp_solver *s, aqp_scalars *sc);
/* Run up to n_iters outer iterations asynchronously (device stops early on a
 * non-finite move); scalars come back with the next aqp_solver_check or
 * aqp_solver_get_scalars. */
int aqp_solver_run(aqp_solver *s, int64_t n_iters);
/* Residuals at (clamp(x), y).  with_rays != 0 additionally forms the window
 * averages and runs the infeasibility tests (a full certification point);
 * with_rays == 0 is the initial / final report (engine.py:373-374,496-497). */
int aqp_solver_check(aqp_solver *s, int with_rays, aqp_check_result *out);
/* state transitions, engine.py:284-333 and the cert bookkeeping of 464-465 */
int aqp_solver_mark_cert(aqp_solver *s);      /* x_last_cert, y_last_cert <- x, y */
int aqp_solver_restart(aqp_solver *s);        /* anchor, round start, z_prev <- x, y  */
int aqp_solver_rollback(aqp_solver *s);       /* x, y, z_prev <- anchor; windows reset  */
int aqp_solver_reset_window(aqp_solver *s);   /* zero window sums, forget avg_prev      */
/* copy out: which: 0 = x_eval (box-projected x), 1 = y, 2 = dual slack r,
 * 3/4 = y-ray candidate 0/1, 5/6 = x-ray candidate 0/1, 7 = x.  A row
 * shard copies its own slice (len = n1-n0 or m1-m0); the host concatenates
 * the ranks' slices in rank order. */
int aqp_solver_read(aqp_solver *s, int which, double *host_out, int64_t len);
/* launches_out[0]: kernels per outer iteration outside the BB loop;
 * launches_out[1]: kernels per BB iteration; launches_out[2]: 1 when the
 * window graph uses programmatic (PDL) edges */
int aqp_solver_counters(aqp_solver *s, int64_t *launches_out);
/* Power iteration for the step size (linalg.py:287-312) on the solver's
 * buffers (call before aqp_solver_init).  *annihilated = 1 when A maps the
 * start vector to 0 (the caller redraws, linalg.py:298-304). */
int aqp_solver_estimate_norm(aqp_solver *s, const double *host_v0, int iters, double *out,
                             int *annihilated);
/* Stand-alone event timing of one hot kernel (bench.py roofline): kernel
 * 0 = BB gradient SpMV pass, 1 = BB step, 2 = P1, 3 = P2 (+fold), 4 = X
 * (+fold), 5 = fold/finalize of pass 0, 6 = dense R x (+ its fold), 7 = dense
 * R'(R x) (dense low-rank problems only); each of `reps`
 * launches follows an L2 flush (streaming read of flush_bytes at flush).  Average
 * device milliseconds per launch in *avg_ms.  Clobbers BB scratch. */
int aqp_solver_time_kernel(aqp_solver *s, int kernel, int reps, void *flush, size_t flush_bytes, double *avg_ms);
/* Device trace, enabled by AQP_TRACE=1 at solver creation: block 0 of every
 * kernel stamps (tag = kind << 32 | grid size, %globaltimer ns); kind 0 SpMV
 * pass, 1 vector pass, 2/3 fold-kernel start/end.  Copies up to `cap` pairs
 * (2*cap words) and resets the ring. */
int aqp_solver_trace(aqp_solver *s, unsigned long long *host_out, int64_t cap, int64_t *count);

/* CUDA IPC of a device buffer (the allocation holding dev_ptr + the offset
 * of dev_ptr in it); handles are 64 bytes. */
int aqp_ipc_get_handle(const void *dev_ptr, void *handle64, size_t *offset);
int aqp_ipc_open(const void *handle64, size_t offset, void **dev_ptr);
int aqp_ipc_close(void *dev_ptr, size_t offset);

#ifdef __cplusplus
}
#endif
#endif /* AQP_H_ */
