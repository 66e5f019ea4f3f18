// aqp_setup.cu -- validation and setup scalars of a device problem, on the device.
//
// The reference's solve starts with host passes over the whole instance:
//   validate(problem)             model.py:181-206 (+ _check_bounds 168-178)
//   default_gamma_sys(problem)    certify.py:167-169 -> QuadOperator.inf_norm_bound
//                                 (linalg.py:218-220, 260-263)
//   finite_bound_scale(con_bounds), |c|_inf   certify.py:54-60
//   QuadOperator.diag_bound()     linalg.py:167-168, 215-216, 252-258
// At C5 (5e8 + 1.25e8 nonzeros) those numpy passes take ~4 s of a ~10 s solve
// call.  Here they are a handful of kernels over the data already in HBM:
//   * flags: NaN / wrong-side infinity / first inverted index of each bound
//     pair, non-finite cost, A values, Q values (the host raises the FIRST
//     violation in the reference's order, with its message);
//   * maxima of non-negative doubles via atomicMax on their bit patterns
//     (exact: max is order-independent);
//   * the abs row / column sums of inf_norm_bound are SEQUENTIAL per row /
//     column in numpy.bincount's order (storage order), so they are bitwise
//     the reference's: the full symmetric Q row i holds the upper triangle's
//     column i (ascending rows, j < i) followed by its row i (j >= i), i.e.
//       col_i = ((0 + |l_0|) + |l_1| + ...) + |U_ii|,  row_i = (0 + |U_ii|) + |u_1| + ...
//     and acc_i = row_i + col_i - |diag_i| (linalg.py:219).
// A row shard computes its rows / columns only; the host combines the ranks'
// structs (max / or / min; R's row sums, which span every rank's columns,
// are then computed on the host).
#include <cuda_runtime.h>

#include <climits>
#include <cstring>

#include "aqp_common.cuh"
#include "aqp_internal.h"

namespace aqp {

namespace {

struct SetupDev {
  int var_nan, var_winf, con_nan, con_winf;
  int cost_bad, a_bad, q_bad, pad;
  unsigned long long var_inv, con_inv;  // first inverted (global) index, ULLONG_MAX: none
  unsigned long long con_scale, cost_inf, q_bound, r_one, r_inf, diag_bound;  // bits of doubles >= +0
};

__device__ __forceinline__ void max_nonneg(unsigned long long *slot, double v) {
  if (!(v > 0.0)) return;  // max(initial=0): zero, -0.0 and negatives never raise it
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

// thread-local max of non-negative doubles as bit patterns; one atomic per
// warp at the end (a per-element atomic on one address serialises in L2:
// ~0.15 s over C5's 1e8 bounds)
struct MaxAcc {
  unsigned long long b = 0;
  __device__ __forceinline__ void add(double v) {
    if (v > 0.0) b = max(b, (unsigned long long)__double_as_longlong(v));
  }
  __device__ __forceinline__ void flush(unsigned long long *slot) {
    unsigned long long x = b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((threadIdx.x & 31) == 0 && x) atomicMax(slot, x);
  }
};

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

// _check_bounds (model.py:168-178) + finite_bound_scale (certify.py:54-60)
__global__ void k_setup_bounds(const double *__restrict__ lo, const double *__restrict__ hi, int64_t n,
                               int64_t base, int *nan_flag, int *winf_flag, unsigned long long *first_inv,
                               unsigned long long *scale) {
  int nan_l = 0, winf_l = 0;
  MaxAcc mx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double l = lo[i], h = hi[i];
    nan_l |= isnan(l) || isnan(h);
    winf_l |= (isinf(l) && l > 0.0) || (isinf(h) && h < 0.0);
    if (l > h) atomicMin(first_inv, (unsigned long long)(base + i));
    if (finite(l)) mx.add(fabs(l));
    if (finite(h)) mx.add(fabs(h));
  }
  if (scale) mx.flush(scale);
  if (__syncthreads_or(nan_l) && threadIdx.x == 0) *nan_flag = 1;
  if (__syncthreads_or(winf_l) && threadIdx.x == 0) *winf_flag = 1;
}

// non-finite flag of an array, and optionally its max |v|
__global__ void k_setup_finite(const double *__restrict__ v, int64_t n, int *bad, unsigned long long *absmax) {
  int b = 0;
  MaxAcc mx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    b |= !finite(x);
    mx.add(fabs(x));
  }
  if (absmax) mx.flush(absmax);
  if (__syncthreads_or(b) && threadIdx.x == 0) *bad = 1;
}

// max(initial=0) of a vector (diag_bound of the diagonal / sparse kinds)
__global__ void k_setup_max(const double *__restrict__ v, int64_t n, unsigned long long *out) {
  MaxAcc mx;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx.add(v[i]);
  mx.flush(out);
}

// SparseQuad.inf_norm_bound (linalg.py:218-220) over the full symmetric rows
// of this problem; also the non-finite flag of Q's values.
__global__ void k_setup_qrows(DevCsr Q, const double *__restrict__ pdiag, int *bad, unsigned long long *out) {
  const int r0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = r0 < Q.rows;
  const int r = live ? r0 : 0;
  const int rg = r + Q.row_off;
  double col = 0.0, row = 0.0;
  bool nonfin = false;
  const int b = Q.ptr[r], e = live ? Q.ptr[r + 1] : b;
  int k = b;
  for (; k < e && Q.idx[k] < rg; ++k) {  // mirrored part: column rg of U, ascending rows
    const double v = Q.val[k];
    nonfin |= !finite(v);
    col += fabs(v);
  }
  if (Q.diag && live) {  // split diagonal (DevCsr::diag): U_ii, last of the column, first of the row
    const double d = Q.diag[r];
    nonfin |= !finite(d);
    col += fabs(d);
    row += fabs(d);
  }
  for (; k < e; ++k) {  // stored part: row rg of U, ascending columns (diagonal first when stored)
    const double v = Q.val[k];
    nonfin |= !finite(v);
    if (Q.idx[k] == rg) col += fabs(v);
    row += fabs(v);
  }
  if (nonfin) *bad = 1;
  MaxAcc mx;
  if (live) mx.add(row + col - fabs(pdiag[r]));
  mx.flush(out);
}

// dense R (k x nl row-major): column abs sums and squares (bincount order:
// ascending rows), max col abs sum and max(p.diag + rsq) (linalg.py:252-263)
__global__ void k_setup_rdense_cols(const double *__restrict__ R, int k, int64_t nl, const double *__restrict__ pdiag,
                                    int *bad, unsigned long long *r_one, unsigned long long *dbound) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = j < nl;
  double ca = 0.0, sq = 0.0;
  bool nonfin = false;
  for (int i = 0; live && i < k; ++i) {
    const double v = R[(int64_t)i * nl + j];
    nonfin |= !finite(v);
    ca += fabs(v);
    sq += v * v;
  }
  if (nonfin) *bad = 1;
  MaxAcc m1, m2;
  if (live) {
    m1.add(ca);
    m2.add(pdiag[j] + sq);
  }
  m1.flush(r_one);
  m2.flush(dbound);
}

// dense R row abs sums: one block per row; the block stages 2048 entries of
// the row in shared memory with coalesced loads, thread 0 adds them in column
// order (the sum stays sequential, the loads do not)
__global__ void __launch_bounds__(256) k_setup_rdense_rows(const double *__restrict__ R, int64_t nl,
                                                           unsigned long long *r_inf) {
  constexpr int kTile = 2048;
  __shared__ double tile[kTile];
  const double *row = R + (int64_t)blockIdx.x * nl;
  double s = 0.0;
  for (int64_t j0 = 0; j0 < nl; j0 += kTile) {
    const int len = (int)(nl - j0 < kTile ? nl - j0 : kTile);
    for (int t = threadIdx.x; t < len; t += blockDim.x) tile[t] = __ldg(row + j0 + t);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int t = 0; t < len; ++t) s += fabs(tile[t]);
    __syncthreads();
  }
  if (threadIdx.x == 0) max_nonneg(r_inf, s);
}

// CSR rows: sequential abs sums (R rows: r_inf; R' rows = R columns: r_one,
// with the squares for diag_bound when pdiag is given)
__global__ void k_setup_csr_rows(DevCsr M, const double *__restrict__ pdiag, int *bad, unsigned long long *absmax,
                                 unsigned long long *dbound) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = r < M.rows;
  double a = 0.0, sq = 0.0;
  bool nonfin = false;
  for (int k = live ? M.ptr[r] : 0, e = live ? M.ptr[r + 1] : 0; k < e; ++k) {
    const double v = M.val[k];
    nonfin |= !finite(v);
    a += fabs(v);
    sq += v * v;
  }
  if (nonfin && bad) *bad = 1;
  MaxAcc m1, m2;
  if (live) {
    m1.add(a);
    if (pdiag) m2.add(pdiag[r] + sq);
  }
  m1.flush(absmax);
  if (pdiag) m2.flush(dbound);
}

inline int grid_n(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

inline double from_bits(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

}  // namespace

}  // namespace aqp

using namespace aqp;

extern "C" {

int aqp_problem_setup_info(aqp_problem *p, aqp_setup_info *out) {
  if (!p || !out) return fail(AQP_EINVAL, "NULL argument");
  cudaStream_t st = p->ctx->stream;
  AQP_CUDA(cudaSetDevice(p->ctx->device));
  static_assert(sizeof(SetupDev) <= 256, "setup_scratch holds SetupDev");
  SetupDev *d = static_cast<SetupDev *>(p->setup_scratch);
  AQP_CUDA(cudaMemsetAsync(d, 0, sizeof(SetupDev), st));
  AQP_CUDA(cudaMemsetAsync(&d->var_inv, 0xff, 2 * sizeof(unsigned long long), st));
  const int64_t nl = p->n1 - p->n0, ml = p->m1 - p->m0;
  if (nl) {
    k_setup_bounds<<<grid_n(nl), 256, 0, st>>>(p->vlo, p->vhi, nl, p->n0, &d->var_nan, &d->var_winf, &d->var_inv,
                                               nullptr);
    k_setup_finite<<<grid_n(nl), 256, 0, st>>>(p->c, nl, &d->cost_bad, &d->cost_inf);
  }
  if (ml)
    k_setup_bounds<<<grid_n(ml), 256, 0, st>>>(p->clo, p->chi, ml, p->m0, &d->con_nan, &d->con_winf, &d->con_inv,
                                               &d->con_scale);
  if (p->A.nnz) k_setup_finite<<<grid_n(p->A.nnz), 256, 0, st>>>(p->A.val, p->A.nnz, &d->a_bad, nullptr);
  int r_inf_done = 1;
  if (p->quad_kind == AQP_QUAD_DIAGONAL) {
    if (nl) {
      k_setup_finite<<<grid_n(nl), 256, 0, st>>>(p->qd, nl, &d->q_bad, nullptr);
      k_setup_max<<<grid_n(nl), 256, 0, st>>>(p->qd, nl, &d->q_bound);  // inf_norm_bound = diag_bound
      k_setup_max<<<grid_n(nl), 256, 0, st>>>(p->qd, nl, &d->diag_bound);
    }
  } else {
    if (p->Q.rows) k_setup_qrows<<<(p->Q.rows + 255) / 256, 256, 0, st>>>(p->Q, p->qd, &d->q_bad, &d->q_bound);
    if (p->quad_kind == AQP_QUAD_SPARSE) {
      if (nl) k_setup_max<<<grid_n(nl), 256, 0, st>>>(p->qd, nl, &d->diag_bound);
    } else if (p->r_dense) {
      const int k = p->R.rows;
      if (nl && k) {
        k_setup_rdense_cols<<<grid_n(nl), 256, 0, st>>>(p->R.val, k, nl, p->qd, &d->q_bad, &d->r_one,
                                                        &d->diag_bound);
        if (p->nranks == 1) k_setup_rdense_rows<<<k, 256, 0, st>>>(p->R.val, nl, &d->r_inf);
      } else if (nl) {
        k_setup_max<<<grid_n(nl), 256, 0, st>>>(p->qd, nl, &d->diag_bound);
      }
      r_inf_done = p->nranks == 1;
    } else {
      // R' rows are R's columns [n0,n1) (stable transpose: ascending rows)
      if (p->Rt.rows)
        k_setup_csr_rows<<<(p->Rt.rows + 255) / 256, 256, 0, st>>>(p->Rt, p->qd, &d->q_bad, &d->r_one,
                                                                    &d->diag_bound);
      if (p->nranks == 1 && p->R.rows)
        k_setup_csr_rows<<<(p->R.rows + 255) / 256, 256, 0, st>>>(p->R, nullptr, nullptr, &d->r_inf, nullptr);
      r_inf_done = p->nranks == 1;
    }
  }
  AQP_CUDA(cudaGetLastError());
  SetupDev h;
  AQP_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  out->var_nan = h.var_nan;
  out->var_wrong_inf = h.var_winf;
  out->con_nan = h.con_nan;
  out->con_wrong_inf = h.con_winf;
  out->var_first_inverted = h.var_inv == ULLONG_MAX ? -1 : (int64_t)h.var_inv;
  out->con_first_inverted = h.con_inv == ULLONG_MAX ? -1 : (int64_t)h.con_inv;
  out->cost_nonfinite = h.cost_bad;
  out->a_nonfinite = h.a_bad;
  out->q_nonfinite = h.q_bad;
  out->r_inf_done = r_inf_done;
  out->con_scale = from_bits(h.con_scale);
  out->cost_inf = from_bits(h.cost_inf);
  out->q_bound = from_bits(h.q_bound);
  out->r_one = from_bits(h.r_one);
  out->r_inf = from_bits(h.r_inf);
  out->diag_bound = from_bits(h.diag_bound);
  return AQP_OK;
}

}  // extern "C"
