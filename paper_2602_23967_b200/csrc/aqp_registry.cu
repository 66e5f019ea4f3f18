// aqp_registry.cu -- host-pointer drop-ins for the reference kernel registry
// (anchorqp/_kernels/__init__.py:16-27, signatures of _core.pyx:29-182).
//
// Each entry point copies its inputs to HBM, runs the sm_100a kernel on the
// calling thread's per-thread stream and copies the result back, exactly the
// contract a ctypes-registered backend needs (inputs borrowed read-only, fresh
// output, deterministic order).  The CSR products use the STRICT plan (one
// thread per row, sequential column order) so they equal the Cython kernels
// bit for bit; the solver itself uses the faster mixed plan.
#include <cstring>
#include <vector>

#include "aqp_common.cuh"
#include "aqp_internal.h"
#include "aqp_kernels.cuh"

namespace aqp {
namespace {

struct DevBuf {
  void *p = nullptr;
  cudaStream_t st;
  explicit DevBuf(cudaStream_t s) : st(s) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 8, st); }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

template <bool S>
struct OpRegStore {
  static constexpr int NS = 0, NM = 0;
  static constexpr bool SYM = S, FINAL = false;
  const double *x;
  double *out;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {}
  __device__ double gather(int c) const { return __ldg(x + c); }
  __device__ void row(int r, double s, RedVals<0, 0> &) const { out[r] = s; }
  __device__ void finalize(const RedVals<0, 0> &) const {}
};

// mode: 0 clamp, 1 cone, 2 diag_prox, 3 natres, 4 dual_step, 5 lincomb3, 6 axpby, 7 support_p
struct OpRegElem {
  static constexpr int NS = 3, NM = 0;
  static constexpr bool FINAL = true;
  int mode;
  const double *a, *b, *c, *lo, *hi;
  const int8_t *codes;
  double s1, s2, s3;
  double *out;
  double *result;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {}
  __device__ void elem(int64_t i, RedVals<3, 0> &acc) const {
    switch (mode) {
      case 0: out[i] = clip(a[i], lo[i], hi[i]); break;
      case 1: out[i] = cone_proj(a[i], codes[i]); break;
      case 2: out[i] = clip((a[i] - s1 * c[i]) / (1.0 + s1 * b[i]), lo[i], hi[i]); break;
      case 3: {
        const double d = a[i] - clip(a[i] - b[i], lo[i], hi[i]);
        acc.s[0] += d * d;
        break;
      }
      case 4: {
        const double w = a[i] / s1 + b[i];
        out[i] = s1 * (w - clip(w, lo[i], hi[i]));
        break;
      }
      case 5: out[i] = s1 * a[i] + s2 * b[i] + s3 * c[i]; break;
      case 6: out[i] = s1 * a[i] + s2 * b[i]; break;
      default: {
        double bad = acc.s[2];
        support_add(a[i], lo[i], hi[i], acc.s[0], acc.s[1], bad);
        acc.s[2] = bad;
      }
    }
  }
  __device__ void finalize(const RedVals<3, 0> &t) const {
    if (mode == 3) *result = t.s[0];
    if (mode == 7) *result = t.s[2] > 0.0 ? INFINITY : t.s[0] + t.s[1];
  }
};

int run_elem_host(int mode, int64_t n, const double *a, const double *b, const double *c, const double *lo,
                  const double *hi, const int8_t *codes, double s1, double s2, double s3, double *out,
                  bool scalar_out) {
  if (n < 0) return fail(AQP_EINVAL, "negative length");
  cudaStream_t st = cudaStreamPerThread;
  const size_t vb = (size_t)n * 8;
  DevBuf da(st), db(st), dc(st), dl(st), dh(st), dk(st), dout(st), dpart(st);
  OpRegElem op{};
  op.mode = mode;
  op.s1 = s1;
  op.s2 = s2;
  op.s3 = s3;
  auto up = [&](DevBuf &d, const void *h, size_t bytes) -> cudaError_t {
    cudaError_t e = d.alloc(bytes);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(d.p, h, bytes, cudaMemcpyHostToDevice, st);
    return e;
  };
  if (a) { AQP_CUDA(up(da, a, vb)); op.a = (const double *)da.p; }
  if (b) { AQP_CUDA(up(db, b, vb)); op.b = (const double *)db.p; }
  if (c) { AQP_CUDA(up(dc, c, vb)); op.c = (const double *)dc.p; }
  if (lo) { AQP_CUDA(up(dl, lo, vb)); op.lo = (const double *)dl.p; }
  if (hi) { AQP_CUDA(up(dh, hi, vb)); op.hi = (const double *)dh.p; }
  if (codes) { AQP_CUDA(up(dk, codes, (size_t)n)); op.codes = (const int8_t *)dk.p; }
  AQP_CUDA(dout.alloc(scalar_out ? 8 : vb));
  op.out = (double *)dout.p;
  op.result = (double *)dout.p;
  const int grid = elem_grid(n);
  AQP_CUDA(dpart.alloc((size_t)grid * kMaxRed * 8 + 256));
  GridRed gr;
  gr.partials = (double *)dpart.p;
  gr.ticket = (unsigned *)((char *)dpart.p + (size_t)grid * kMaxRed * 8);
  AQP_CUDA(cudaMemsetAsync(gr.ticket, 0, 64, st));
  elem_op<OpRegElem><<<grid, kThreads, 0, st>>>(n, op, gr);
  AQP_CUDA(cudaGetLastError());
  AQP_CUDA(cudaMemcpyAsync(out, dout.p, scalar_out ? 8 : vb, cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  return AQP_OK;
}

// kind 0: A x; 1: A' x; 2: sym(upper) x
int run_csr_host(int kind, const int64_t *indptr, const int64_t *indices, const double *data, const double *x,
                 int64_t nrows, int64_t ncols, double *out) {
  if (nrows < 0 || ncols < 0) return fail(AQP_EINVAL, "negative dimension");
  const int64_t nnz = indptr[nrows];
  if (nnz >= INT32_MAX / 4 || nrows >= INT32_MAX || ncols >= INT32_MAX)
    return fail(AQP_ERANGE, "matrix exceeds int32 device indexing");
  cudaStream_t st = cudaStreamPerThread;
  aqp_ctx ctx;
  ctx.stream = st;
  cudaGetDevice(&ctx.device);
  DevBuf dptr(st), didx(st), dval(st), dx(st), dout(st), store(st), scratch(st), dbad(st);
  AQP_CUDA(dptr.alloc((nrows + 1) * 8));
  AQP_CUDA(didx.alloc(nnz * 8));
  AQP_CUDA(dval.alloc(nnz * 8));
  AQP_CUDA(cudaMemcpyAsync(dptr.p, indptr, (nrows + 1) * 8, cudaMemcpyHostToDevice, st));
  if (nnz) {
    AQP_CUDA(cudaMemcpyAsync(didx.p, indices, nnz * 8, cudaMemcpyHostToDevice, st));
    AQP_CUDA(cudaMemcpyAsync(dval.p, data, nnz * 8, cudaMemcpyHostToDevice, st));
  }
  const int64_t xlen = kind == 1 ? nrows : ncols;
  const int64_t olen = kind == 1 ? ncols : nrows;
  AQP_CUDA(dx.alloc(xlen * 8));
  if (xlen) AQP_CUDA(cudaMemcpyAsync(dx.p, x, xlen * 8, cudaMemcpyHostToDevice, st));
  AQP_CUDA(dout.alloc(olen * 8));
  AQP_CUDA(dbad.alloc(64));
  AQP_CUDA(cudaMemsetAsync(dbad.p, 0, 64, st));
  // storage for the source CSR and its transpose / symmetric expansion
  Bump lay;
  CsrStore s0, s1;
  layout_csr(lay, s0, nrows, nnz);
  layout_csr(lay, s1, kind == 1 ? ncols : nrows, kind == 2 ? 2 * nnz : nnz);
  AQP_CUDA(store.alloc(lay.used + 256));
  Bump b;
  b.base = store.p;
  b.cap = lay.used + 256;
  layout_csr(b, s0, nrows, nnz);
  layout_csr(b, s1, kind == 1 ? ncols : nrows, kind == 2 ? 2 * nnz : nnz);
  DevCsr M0, M1;
  AQP_TRY(upload_csr(&ctx, s0, M0, nrows, ncols, (const int64_t *)dptr.p, (const int64_t *)didx.p,
                     (const double *)dval.p, nnz, indptr, true, (int *)dbad.p));
  GridRed gr{};
  const DevCsr *M = &M0;
  if (kind != 0) {
    const size_t sb = kind == 1 ? transpose_scratch_bytes(nnz, ncols) : symmetrize_scratch_bytes(nnz, nrows);
    AQP_CUDA(scratch.alloc(sb));
    Bump sc;
    sc.base = scratch.p;
    sc.cap = sb;
    if (kind == 1) {
      AQP_TRY(transpose_csr(&ctx, M0, s1, M1, true, sc));
    } else {
      int64_t nf = 0;
      AQP_TRY(symmetrize_csr(&ctx, M0, s1, M1, true, sc, &nf));
    }
    M = &M1;
  }
  if (kind == 2) {
    OpRegStore<true> op{(const double *)dx.p, (double *)dout.p};
    spmv_op<OpRegStore<true>><<<M->nitems, kThreads, M->smem_bytes, st>>>(*M, op, gr);
  } else {
    OpRegStore<false> op{(const double *)dx.p, (double *)dout.p};
    spmv_op<OpRegStore<false>><<<M->nitems, kThreads, M->smem_bytes, st>>>(*M, op, gr);
  }
  AQP_CUDA(cudaGetLastError());
  int bad = 0;
  AQP_CUDA(cudaMemcpyAsync(&bad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (olen) AQP_CUDA(cudaMemcpyAsync(out, dout.p, olen * 8, cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(AQP_EINVAL, "column index out of range");
  return AQP_OK;
}

}  // namespace
}  // namespace aqp

using namespace aqp;

extern "C" {

int aqp_csr_matvec(const int64_t *indptr, const int64_t *indices, const double *data, const double *x,
                   int64_t nrows, int64_t ncols, double *out) {
  return run_csr_host(0, indptr, indices, data, x, nrows, ncols, out);
}

int aqp_csr_matvec_t(const int64_t *indptr, const int64_t *indices, const double *data, const double *x,
                     int64_t nrows, int64_t ncols, double *out) {
  return run_csr_host(1, indptr, indices, data, x, nrows, ncols, out);
}

int aqp_sym_matvec(const int64_t *indptr, const int64_t *indices, const double *data, const double *diag,
                   const double *x, int64_t n, double *out) {
  (void)diag;  // the Cython kernel reads stored entries only (_core.pyx:62-80)
  return run_csr_host(2, indptr, indices, data, x, n, n, out);
}

int aqp_clamp(const double *x, const double *lo, const double *hi, int64_t n, double *out) {
  return run_elem_host(0, n, x, nullptr, nullptr, lo, hi, nullptr, 0, 0, 0, out, false);
}

int aqp_cone_project(const double *z, const int8_t *codes, int64_t n, double *out) {
  return run_elem_host(1, n, z, nullptr, nullptr, nullptr, nullptr, codes, 0, 0, 0, out, false);
}

int aqp_diag_prox_step(const double *xk, const double *q, const double *linear, double tau, const double *lo,
                       const double *hi, int64_t n, double *out) {
  return run_elem_host(2, n, xk, q, linear, lo, hi, nullptr, tau, 0, 0, out, false);
}

int aqp_natural_res_sq(const double *x, const double *g, const double *lo, const double *hi, int64_t n,
                       double *out) {
  return run_elem_host(3, n, x, g, nullptr, lo, hi, nullptr, 0, 0, 0, out, true);
}

int aqp_dual_step(const double *y, const double *ax, double sigma, const double *lo, const double *hi, int64_t m,
                  double *out) {
  return run_elem_host(4, m, y, ax, nullptr, lo, hi, nullptr, sigma, 0, 0, out, false);
}

int aqp_lincomb3(double a, const double *x, double b, const double *y, double c, const double *z, int64_t n,
                 double *out) {
  return run_elem_host(5, n, x, y, z, nullptr, nullptr, nullptr, a, b, c, out, false);
}

int aqp_axpby(double a, const double *x, double b, const double *y, int64_t n, double *out) {
  return run_elem_host(6, n, x, y, nullptr, nullptr, nullptr, nullptr, a, b, 0, out, false);
}

int aqp_support_p(const double *z, const double *lo, const double *hi, int64_t n, double *out) {
  return run_elem_host(7, n, z, nullptr, nullptr, lo, hi, nullptr, 0, 0, 0, out, true);
}

}  // extern "C"
