// aqp_scale.cu -- device-side Ruiz / Pock-Chambolle equilibration of a
// problem (BASELINE.json north star; absent from the reference, so it is
// opt-in and off by default: SolverParams.scaling).
//
// The KKT matrix K = [[Q, A'], [A, 0]] is scaled as diag(D, E) K diag(D, E):
//   Ruiz (iters rounds):   D_j /= sqrt(max(|Q~|_inf col j, |A~|_inf col j)),
//                          E_r /= sqrt(|A~|_inf row r)
//   Pock-Chambolle (a=1):  the same with l1 norms, once after Ruiz.
// Column norms come from the row passes of the explicit transposes (A' rows
// are A's columns; the full symmetric Q is its own transpose), one thread per
// row, so no atomics.  Then, in place on the device problem:
//   A~ = E A D, A'~ = D A' E, Q~ = D Q D (R~ = R D), c~ = D c,
//   l_v~ = l_v / D, u_v~ = u_v / D, l_c~ = E l_c, u_c~ = E u_c.
// The solve runs on the scaled problem; the host unscales iterates (x = D x~,
// y = E y~) into a second, unscaled solver for every certification point, so
// termination and certificates are the reference's, on the original problem.
#include <cmath>

#include "aqp_common.cuh"
#include "aqp_internal.h"
#include "aqp_kernels.cuh"

namespace aqp {

// out[r] = max_k |val_k| * rs[r] * cs[col_k]  (l1: sum instead of max)
__global__ void k_row_norm(DevCsr M, const double *__restrict__ rs, const double *__restrict__ cs, int l1,
                           double *__restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M.rows) return;
  double a = 0.0;
  const double s = rs[r];
  for (int k = M.ptr[r]; k < M.ptr[r + 1]; ++k) {
    const double v = fabs(M.val[k]) * s * cs[M.idx[k]];
    a = l1 ? a + v : fmax(a, v);
  }
  out[r] = a;
}

// d *= 1 / sqrt(max(n1, n2)) (or the sum for l1); zero norms leave d alone
__global__ void k_update(double *__restrict__ d, const double *__restrict__ n1, const double *__restrict__ n2,
                         int64_t n, int l1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = n1[i];
  if (n2) a = l1 ? a + n2[i] : fmax(a, n2[i]);
  if (a > 0.0 && isfinite(a)) d[i] /= sqrt(a);
}

__global__ void k_scale_csr(DevCsr M, const double *__restrict__ rs, const double *__restrict__ cs,
                            double *__restrict__ val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M.rows) return;
  const double s = rs[r];
  for (int k = M.ptr[r]; k < M.ptr[r + 1]; ++k) val[k] = val[k] * s * cs[M.idx[k]];
}

// the SELL-32 copy of a uniform plan's matrix (DevCsr::sell_*) follows its CSR
// (thread = SELL position: natural SELL position p is row p; SELL-P position
// p is row (p & ~255) + sell_perm[p], and long rows are not in the slices)
__global__ void k_scale_sell(DevCsr M, const double *__restrict__ rs, const double *__restrict__ cs, bool pair) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M.rows || !M.sell_val) return;
  const int r = M.sell_perm ? (p & ~255) + M.sell_perm[p] : p;
  const int len = M.ptr[r + 1] - M.ptr[r];
  if (M.sell_perm && len > kThreadRowMax) return;
  const int64_t off0 = M.sell_off[p >> 5];
  const int lane = p & 31;
  double *sval = const_cast<double *>(M.sell_val);
  const double s = rs[r];
  for (int k = 0; k < len; ++k) {
    const int64_t q = sell_pos(off0, lane, k, pair);
    sval[q] = sval[q] * s * cs[M.sell_idx[q]];
  }
}

__global__ void k_scale_dense(double *__restrict__ R, int k, int64_t n, const double *__restrict__ cs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)k * n) return;
  R[t] *= cs[t % n];
}

// vectors: c *= D, qd *= D^2, var bounds /= D, con bounds *= E
__global__ void k_scale_vec(double *c, double *qd, double *vlo, double *vhi, const double *D, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = D[i];
  c[i] *= d;
  qd[i] *= d * d;
  vlo[i] /= d;  // +-inf stay infinite
  vhi[i] /= d;
}
__global__ void k_scale_con(double *clo, double *chi, const double *E, int64_t m) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  clo[i] *= E[i];
  chi[i] *= E[i];
}
__global__ void k_diag_norm(const double *__restrict__ q, const double *__restrict__ D, int64_t n,
                            double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fabs(q[i]) * D[i] * D[i];
}
// a split-out diagonal of Q (DevCsr::diag) joins the row norm / is scaled by D^2
// row norms of a full symmetric Q whose diagonal is split out of the CSR
// (DevCsr::diag): the diagonal term enters at its column position, so the l1
// sums are bitwise those of the unsplit CSR (AQP_SPLIT_DIAG=0)
__global__ void k_row_norm_split(DevCsr M, const double *__restrict__ D, int l1, double *__restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M.rows) return;
  const int gr = r + M.row_off;
  const double s = D[r];
  const double dv = fabs(M.diag[r]) * s * D[r];
  double a = 0.0;
  bool done = false;
  for (int k = M.ptr[r]; k < M.ptr[r + 1]; ++k) {
    if (!done && M.idx[k] > gr) {
      a = l1 ? a + dv : fmax(a, dv);
      done = true;
    }
    const double v = fabs(M.val[k]) * s * D[M.idx[k]];
    a = l1 ? a + v : fmax(a, v);
  }
  if (!done) a = l1 ? a + dv : fmax(a, dv);
  out[r] = a;
}
// q = (q * d) * d: the order k_scale_csr applies to a CSR diagonal entry
__global__ void k_scale_diag(double *q, const double *D, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) q[i] = q[i] * D[i] * D[i];
}
__global__ void k_fill(double *p, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

inline unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>((n + 255) / 256, 1); }

}  // namespace aqp

using namespace aqp;

extern "C" {

int aqp_problem_scale(aqp_problem *p, int ruiz_iters, int pock_chambolle, double *D, double *E, void *scratch,
                      size_t scratch_bytes) {
  if (!p || !D || !E) return fail(AQP_EINVAL, "NULL argument");
  if (p->nranks > 1) return fail(AQP_EINVAL, "scale before sharding / not with row shards");
  const int64_t n = p->n, m = p->m;
  if ((size_t)(2 * n + m) * 8 > scratch_bytes) return fail(AQP_ENOMEM, "scaling scratch too small");
  cudaStream_t st = p->ctx->stream;
  double *nx1 = static_cast<double *>(scratch), *nx2 = nx1 + n, *ny = nx2 + n;
  k_fill<<<grid_of(n), 256, 0, st>>>(D, n, 1.0);
  k_fill<<<grid_of(m), 256, 0, st>>>(E, m, 1.0);
  const bool sparse_q = p->quad_kind != AQP_QUAD_DIAGONAL;
  const bool lowrank = p->quad_kind == AQP_QUAD_SPARSE_LOW_RANK;
  for (int round = 0; round < ruiz_iters + (pock_chambolle ? 1 : 0); ++round) {
    const int l1 = round >= ruiz_iters;  // the Pock-Chambolle pass uses l1 norms
    // x side: A' rows (= A columns) with row scale D, col scale E
    if (n) k_row_norm<<<grid_of(n), 256, 0, st>>>(p->At, D, E, l1, nx1);
    if (sparse_q && n) {
      if (p->Q.diag)  // full symmetric P: rows = columns
        k_row_norm_split<<<grid_of(n), 256, 0, st>>>(p->Q, D, l1, nx2);
      else
        k_row_norm<<<grid_of(n), 256, 0, st>>>(p->Q, D, D, l1, nx2);
    } else if (n) {
      k_diag_norm<<<grid_of(n), 256, 0, st>>>(p->qd, D, n, nx2);    // diagonal Q: |q_j| d_j^2
    }
    if (m) k_row_norm<<<grid_of(m), 256, 0, st>>>(p->A, E, D, l1, ny);
    AQP_CUDA(cudaGetLastError());
    // combine: x norm = max / sum of the A' and Q parts
    if (n) k_update<<<grid_of(n), 256, 0, st>>>(D, nx1, nx2, n, l1);
    if (m) k_update<<<grid_of(m), 256, 0, st>>>(E, ny, nullptr, m, l1);
    AQP_CUDA(cudaGetLastError());
  }
  // apply in place (CSR values, and the SELL copies of uniform plans)
  if (m) k_scale_csr<<<grid_of(m), 256, 0, st>>>(p->A, E, D, const_cast<double *>(p->A.val));
  if (n) k_scale_csr<<<grid_of(n), 256, 0, st>>>(p->At, D, E, const_cast<double *>(p->At.val));
  if (sparse_q && n) k_scale_csr<<<grid_of(n), 256, 0, st>>>(p->Q, D, D, const_cast<double *>(p->Q.val));
  if (sparse_q && n && p->Q.diag) k_scale_diag<<<grid_of(n), 256, 0, st>>>(const_cast<double *>(p->Q.diag), D, n);
  if (m && p->A.sell_val) k_scale_sell<<<grid_of(m), 256, 0, st>>>(p->A, E, D, true);
  if (n && p->At.sell_val) k_scale_sell<<<grid_of(n), 256, 0, st>>>(p->At, D, E, true);
  if (sparse_q && n && p->Q.sell_val) k_scale_sell<<<grid_of(n), 256, 0, st>>>(p->Q, D, D, false);
  if (lowrank) {
    if (p->r_dense) {
      k_scale_dense<<<grid_of((int64_t)p->R.rows * n), 256, 0, st>>>(const_cast<double *>(p->R.val), p->R.rows, n, D);
    } else {
      // R (k x n): columns by D; R' (n x k): rows by D (nx1 holds k ones)
      if (p->R.rows > n) return fail(AQP_EINVAL, "low-rank factor with more rows than columns");
      k_fill<<<grid_of(std::max<int64_t>(p->R.rows, 1)), 256, 0, st>>>(nx1, std::max<int64_t>(p->R.rows, 1), 1.0);
      k_scale_csr<<<grid_of(p->R.rows), 256, 0, st>>>(p->R, nx1, D, const_cast<double *>(p->R.val));
      k_scale_csr<<<grid_of(n), 256, 0, st>>>(p->Rt, D, nx1, const_cast<double *>(p->Rt.val));
      if (p->R.sell_val) k_scale_sell<<<grid_of(p->R.rows), 256, 0, st>>>(p->R, nx1, D, true);
      if (p->Rt.sell_val) k_scale_sell<<<grid_of(n), 256, 0, st>>>(p->Rt, D, nx1, true);
    }
  }
  if (n) k_scale_vec<<<grid_of(n), 256, 0, st>>>(p->c, p->qd, p->vlo, p->vhi, D, n);
  if (m) k_scale_con<<<grid_of(m), 256, 0, st>>>(p->clo, p->chi, E, m);
  AQP_CUDA(cudaGetLastError());
  AQP_CUDA(cudaStreamSynchronize(st));
  return AQP_OK;
}

}  // extern "C"
