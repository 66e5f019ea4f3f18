// aqp_internal.h -- library-private structs shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include <mutex>

#include "aqp_common.cuh"

// bump allocator over a caller-provided workspace; with base == nullptr it
// only measures (the "sizes" dry run uses the very same layout code)
namespace aqp {
struct Bump {
  void *base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  bool overflow = false;
  void *take(size_t bytes);
};

struct CsrStore {
  int *ptr = nullptr;
  int *idx = nullptr;
  double *val = nullptr;
  int64_t cap_nnz = 0;
  PlanItem *plan = nullptr;
  int64_t plan_cap = 0;
  double *seg_part = nullptr;
  unsigned *seg_ticket = nullptr;
  int64_t seg_cap = 0;
  int64_t *sell_off = nullptr;  // SELL-32 slice offsets (8 per 256-row block + 2), planned by plan_sell
  uint8_t *sell_perm = nullptr;  // SELL-P position -> row within its 256-row block (rows bytes)
};

void layout_csr(Bump &b, CsrStore &s, int64_t rows, int64_t nnz);
int upload_csr(aqp_ctx *ctx, CsrStore &s, DevCsr &M, int64_t rows, int64_t cols, const int64_t *d_ptr,
               const int64_t *d_idx, const double *d_val, int64_t nnz, const int64_t *host_ptr, bool strict,
               int *d_bad);
int transpose_csr(aqp_ctx *ctx, const DevCsr &src, CsrStore &t, DevCsr &T, bool strict, Bump &scratch,
                  int64_t col0 = 0, int64_t col1 = -1, int64_t row_base = 0, int64_t out_cols = -1,
                  bool *deferred = nullptr);
int plan_deferred_at(aqp_problem *p);
int symmetrize_csr(aqp_ctx *ctx, const DevCsr &U, CsrStore &f, DevCsr &F, bool strict, Bump &scratch,
                   int64_t *nfull_out, int64_t row_base = 0, int64_t r0 = 0, int64_t r1 = -1);
size_t transpose_scratch_bytes(int64_t nnz, int64_t cols);
// synchronous staged host <-> device copy (aqp_xfer.cu)
int bulk_copy(int device, void *dev, void *host, size_t bytes, bool h2d);
int xfer_init(int device);
size_t symmetrize_scratch_bytes(int64_t nnz, int64_t n);
}  // namespace aqp

struct aqp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  // pinned host staging shared by every solver of this (device, stream):
  // allocated once (cudaMallocHost / cudaFreeHost synchronise the device, so
  // they must not run per solve while other streams work), used in stream order
  void *pinned = nullptr;
  void *bounce = nullptr;
  unsigned ring_i = 0;
  // every solver call on this context holds it: solvers of one (device,
  // stream) share the pinned control ring, pull block and bounce buffer, and
  // host threads may call concurrently (ctypes releases the GIL)
  std::recursive_mutex mu;
};

struct aqp_problem {
  aqp_ctx *ctx = nullptr;
  int64_t n = 0, m = 0;
  int quad_kind = 0;
  aqp::CsrStore sA, sAt, sQ, sR, sRt;
  aqp::DevCsr A, At, Q, R, Rt;
  int64_t q_full_nnz = 0;
  int64_t sell_total[5] = {};  // padded SELL-32 entries of A, A', Q, R, R' (0: no SELL copy)
  bool sell_sorted[5] = {};    // ... in the SELL-P (block-sorted) layout
  // A' planned lazily: a staged (non-uniform) A' that gets the SELL-P layout
  // never runs its CSR plan, so the host planning pass (0.12 s on C5's 5e7
  // rows) waits until a solver needs it without SELL-P (plan_deferred_at)
  bool at_plan_deferred = false;
  int r_dense = 0;  // R held dense row-major in R.val (R.rows x n); no R' CSR
  double *qdiag = nullptr;  // Q's diagonal when split out of its CSR (DevCsr::diag)
  double *c = nullptr, *vlo = nullptr, *vhi = nullptr, *qd = nullptr, *clo = nullptr, *chi = nullptr;
  int8_t *cone_r = nullptr, *recc_x = nullptr, *cone_y = nullptr, *recc_s = nullptr;
  int *bad = nullptr;
  void *setup_scratch = nullptr;  // 256 B of device memory for aqp_problem_setup_info
  aqp_problem_info info{};
  // row shard (aqp_shard_desc): this rank stores rows [n0,n1) of A' / Q and
  // [m0,m1) of A only; gathered vectors live in the windows xwin / ywin
  // (every rank's, [lo, hi) pairs), sized by the max-over-ranks capacities so
  // the peer-visible solver layout is identical on every rank
  int rank = 0, nranks = 1;
  int64_t n0 = 0, n1 = 0, m0 = 0, m1 = 0;
  int64_t xwin[2 * aqp::kMaxRanks] = {}, ywin[2 * aqp::kMaxRanks] = {};
  int64_t nl_cap = 0, ml_cap = 0, xw_cap = 0, yw_cap = 0;
  int64_t xw0() const { return xwin[2 * rank]; }
  int64_t yw0() const { return ywin[2 * rank]; }
};
