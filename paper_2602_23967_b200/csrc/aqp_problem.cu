// aqp_problem.cu -- context, device problem upload and the SpMV work planner.
//
// Device layout of a problem (all in one caller-provided persistent workspace):
//   A   : m x n CSR, int32 ptr/idx, f64 val                 (reference linalg.py:28-112)
//   A'  : n x m CSR built on the device by a STABLE radix sort of A's entries
//         by column -- entries of a column keep ascending row order, so the
//         row-sequential A' product reproduces the Cython scatter order of
//         _core.pyx:45-59 bit for bit, with no atomics.
//   Q   : n x n full symmetric CSR expanded from the upper triangle
//         (linalg.py:177-227); each row is [mirrored lower part | stored upper
//         part] in ascending column order, again via one stable sort.
//   R, R' (low-rank kind): k x n CSR and its transpose (linalg.py:230-266).
//   c, l_v, u_v, l_c, u_c; int8 cone codes (model.py:85-112) built on device.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "aqp_common.cuh"
#include "aqp_internal.h"

namespace aqp {

// AQP_TIMING=1: stream-synchronised wall time of each setup step of
// aqp_problem_create, printed to stderr (diagnostics only; off by default)
static void step_mark(cudaStream_t st, const char *what) {
  static const bool on = [] {
    const char *e = getenv("AQP_TIMING");
    return e && e[0] == '1';
  }();
  static auto t = std::chrono::steady_clock::now();
  if (!on) return;
  cudaStreamSynchronize(st);
  const auto now = std::chrono::steady_clock::now();
  if (what) fprintf(stderr, "AQP_TIMING %s %.4f\n", what, std::chrono::duration<double>(now - t).count());
  t = now;
}
struct StepTimer {
  cudaStream_t st;
  explicit StepTimer(cudaStream_t s) : st(s) { step_mark(st, nullptr); }
  void operator()(const char *what) { step_mark(st, what); }
};

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  set_error(msg);
  return code;
}

// ---------------------------------------------------------------- bump allocator
void *Bump::take(size_t bytes) {
  size_t off = (used + 255) & ~size_t(255);
  used = off + bytes;
  if (base == nullptr) return nullptr;
  if (used > cap) {
    overflow = true;
    return nullptr;
  }
  return static_cast<char *>(base) + off;
}

// ---------------------------------------------------------------- planner
template <class P>
static std::vector<PlanItem> plan_rows(const P *ptr, int64_t rows, bool strict, int *nlongseg, bool staged) {
  std::vector<PlanItem> items;
  int segs = 0;
  int64_t i = 0;
  while (i < rows) {
    const int64_t len = (int64_t)(ptr[i + 1] - ptr[i]);
    if (len > kTileNnz && strict) {
      PlanItem it{};
      it.row0 = (int)i;
      it.row1 = (int)i + 1;
      it.k0 = (int)ptr[i];
      it.k1 = (int)ptr[i + 1];
      it.kind = kItemLongSeq;
      it.nseg = 1;
      items.push_back(it);
      ++i;
      continue;
    }
    if (len > kTileNnz) {
      const int nseg = (int)((len + kSegNnz - 1) / kSegNnz);
      for (int s = 0; s < nseg; ++s) {
        PlanItem it{};
        it.row0 = (int)i;
        it.row1 = (int)i + 1;
        it.k0 = (int)(ptr[i] + (int64_t)s * kSegNnz);
        it.k1 = (int)std::min<int64_t>(ptr[i] + (int64_t)(s + 1) * kSegNnz, ptr[i + 1]);
        it.kind = kItemLong;
        it.seg = s;
        it.nseg = nseg;
        it.segbase = segs;
        items.push_back(it);
      }
      segs += nseg;
      ++i;
      continue;
    }
    // THREAD item: up to 256 consecutive rows of <= kThreadRowMax nonzeros,
    // one thread per row, sequential in column order (no shared memory)
    const int64_t row_max = strict ? (int64_t)kTileNnz : (int64_t)kThreadRowMax;
    const int64_t start = i;
    if (staged) {  // STAGED item: <= 256 short rows whose nonzeros fit one tile
      while (i < rows && i - start < kThreads && (int64_t)(ptr[i + 1] - ptr[i]) <= row_max &&
             (int64_t)(ptr[i + 1] - ptr[start]) <= (int64_t)kTileNnz)
        ++i;
    } else {
      while (i < rows && i - start < kThreads && (int64_t)(ptr[i + 1] - ptr[i]) <= row_max) ++i;
    }
    if (i > start) {
      PlanItem it{};
      it.row0 = (int)start;
      it.row1 = (int)i;
      it.k0 = (int)ptr[start];
      it.k1 = (int)ptr[i];
      it.kind = staged ? kItemStaged : kItemThread;
      items.push_back(it);
      continue;
    }
    // WARP item: medium rows staged in shared memory (<= kTileNnz per tile)
    int64_t nnz = 0;
    while (i < rows && i - start < kThreads) {
      const int64_t l = (int64_t)(ptr[i + 1] - ptr[i]);
      if (l <= row_max || l > kTileNnz || nnz + l > kTileNnz) break;
      nnz += l;
      ++i;
    }
    PlanItem it{};
    it.row0 = (int)start;
    it.row1 = (int)i;
    it.k0 = (int)ptr[start];
    it.k1 = (int)ptr[i];
    it.kind = kItemWarp;
    items.push_back(it);
  }
  if (items.empty()) {  // zero rows: one empty item so fused finalizers still run
    PlanItem it{};
    it.kind = kItemThread;
    items.push_back(it);
  }
  *nlongseg = segs;
  return items;
}

int64_t plan_capacity(int64_t rows, int64_t nnz) {
  // THREAD/WARP items break only at 256 rows, at a row-length class change
  // or a full tile; long rows add their segments
  return 2 * (rows / kThreads) + 2 * (nnz / kThreadRowMax) + 3 * (nnz / kTileNnz) + nnz / kSegNnz + 16;
}

// ---------------------------------------------------------------- setup kernels
__global__ void k_i64_to_i32(const int64_t *__restrict__ in, int *__restrict__ out, int64_t n,
                             int64_t limit, int *bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v > limit) *bad = 1;
    out[i] = (int)v;
  }
}

__global__ void k_row_ids(const int *__restrict__ ptr, int rows, int *__restrict__ rid) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) rid[k] = r;
}

__global__ void k_iota(int *out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int)i;
}

// Key counts from the SORTED keys (counts zeroed): a run [i, j] of key k adds
// j + 1 - i, as two atomics at its ends -- two per distinct key instead of one
// per entry (C5's A': 1e8 instead of 5e8 scattered atomics, 21 -> ~2 ms)
__global__ void k_run_counts(const int *__restrict__ s, int64_t n, int *counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = s[i];
    if (i == 0 || s[i - 1] != k) atomicSub(counts + k, (int)i);
    if (i == n - 1 || s[i + 1] != k) atomicAdd(counts + k, (int)(i + 1));
  }
}

// transpose keys restricted to the column window [col0, col1): an entry
// outside it gets the sentinel key col1 - col0 (sorted last, then dropped)
__global__ void k_tkeys(const int *__restrict__ idx, int64_t nnz, int col0, int col1, int *__restrict__ keys) {
  const int sent = col1 - col0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int c = idx[k];
    keys[k] = (c >= col0 && c < col1) ? c - col0 : sent;
  }
}

// transpose gather: out entry p comes from source entry src[p]; its column
// is the source row, offset by row_base (global row of a block's row 0)
__global__ void k_gather_t(const int *__restrict__ src, const int *__restrict__ rid,
                           const double *__restrict__ val, int64_t n, int row_base, int *__restrict__ out_idx,
                           double *__restrict__ out_val) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int k = src[p];
    out_idx[p] = row_base + rid[k];
    out_val[p] = val[k];
  }
}

// ptr[i] = src[r0 + i] - src[r0] (a row window of a CSR, rebased)
__global__ void k_rebase_ptr(const int *__restrict__ src, int64_t r0, int64_t rows, int *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[r0 + i] - src[r0];
}

// full-symmetric expansion of an upper-triangle block whose row 0 is global
// row `row_base`, restricted to the output rows [r0, r1); the combined entry
// list is
//   [0, nnz)      mirrored copies (row = col_k, col = row_k), diagonal -> sentinel
//   [nnz, 2nnz)   the stored upper entries (row = row_k, col = col_k)
// with key = output row - r0, or the sentinel r1 - r0 for entries outside
// the output rows (sorted last, then dropped).
__global__ void k_sym_keys(const int *__restrict__ rid, const int *__restrict__ col, int64_t nnz, int row_base,
                           int r0, int r1, int *__restrict__ keys) {
  const int sent = r1 - r0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int r = row_base + rid[k], c = col[k];
    keys[k] = (c == r || c < r0 || c >= r1) ? sent : c - r0;
    keys[nnz + k] = (r >= r0 && r < r1) ? r - r0 : sent;
  }
}

__global__ void k_sym_gather(const int *__restrict__ src, const int *__restrict__ rid,
                             const int *__restrict__ col, const double *__restrict__ val, int64_t nnz,
                             int64_t nfull, int row_base, int *__restrict__ out_idx, double *__restrict__ out_val) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nfull; p += (int64_t)gridDim.x * blockDim.x) {
    const int s = src[p];
    if (s < nnz) {  // mirrored: column is the source row
      out_idx[p] = row_base + rid[s];
      out_val[p] = val[s];
    } else {
      out_idx[p] = col[s - nnz];
      out_val[p] = val[s - nnz];
    }
  }
}

// cone tables of model.py:85-112 indexed by (lower finite)*2 + (upper finite)
__global__ void k_cones(const double *__restrict__ lo, const double *__restrict__ hi, int64_t n,
                        int8_t *__restrict__ dual, int8_t *__restrict__ recc, int dual_is_y) {
  // dual_y: (F,F)->ZERO (F,T)->NONNEG (T,F)->NONPOS (T,T)->FREE
  // dual_r: (F,F)->ZERO (F,T)->NONPOS (T,F)->NONNEG (T,T)->FREE
  // recession: (F,F)->FREE (F,T)->NONPOS (T,F)->NONNEG (T,T)->ZERO
  const int8_t ty[4] = {AQP_ZERO, AQP_NONNEG, AQP_NONPOS, AQP_FREE};
  const int8_t tr[4] = {AQP_ZERO, AQP_NONPOS, AQP_NONNEG, AQP_FREE};
  const int8_t tc[4] = {AQP_FREE, AQP_NONPOS, AQP_NONNEG, AQP_ZERO};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (isfinite(lo[i]) ? 2 : 0) + (isfinite(hi[i]) ? 1 : 0);
    dual[i] = dual_is_y ? ty[p] : tr[p];
    recc[i] = tc[p];
  }
}

static inline int setup_grid(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

// ---------------------------------------------------------------- CSR upload / transpose
static size_t sort_temp_bytes(int64_t n_items) {
  size_t a = 0, b = 0;
  if (n_items <= 0) n_items = 1;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const int *)nullptr, (int *)nullptr, (const int *)nullptr,
                                  (int *)nullptr, (int)n_items);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int *)nullptr, (int *)nullptr, (int)n_items + 1);
  return std::max(a, b);
}

static int to_i32(const int64_t *in, int *out, int64_t n, int64_t limit, int *d_bad, cudaStream_t st) {
  if (n == 0) return AQP_OK;
  k_i64_to_i32<<<setup_grid(n), 256, 0, st>>>(in, out, n, limit, d_bad);
  AQP_CUDA(cudaGetLastError());
  return AQP_OK;
}

// ptr: (rows+1) counts -> exclusive scan; keys sorted stably
static int counts_to_ptr(int *counts, int rows, int *ptr_out, void *tmp, size_t tmp_bytes, cudaStream_t st) {
  size_t need = tmp_bytes;
  AQP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, counts, ptr_out, rows + 1, st));
  return AQP_OK;
}

// SELL-32 copy of a uniform plan's matrix (DevCsr::sell_*): library-owned
// device memory, released by free_sell (problem destroy / re-plan).
__global__ void k_fill_sell(const int *__restrict__ ptr, const int *__restrict__ idx, const double *__restrict__ val,
                            int rows, const int64_t *__restrict__ off, int *sidx, double *sval, bool pair) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int b = ptr[r], e = ptr[r + 1];
  const int64_t off0 = off[r >> 5];
  const int lane = r & 31;
  for (int k = 0; k < e - b; ++k) {
    sidx[sell_pos(off0, lane, k, pair)] = idx[b + k];
    sval[sell_pos(off0, lane, k, pair)] = val[b + k];
  }
}

// Column window of each rt-row group (spmv_ring_op): [min, max] column
// of its nonzeros, and its own rows when a split diagonal gathers x[row].
__global__ void k_win_range(const int *__restrict__ ptr, const int *__restrict__ idx, int rows, int rt, bool own,
                            int2 *win) {
  const int r0 = blockIdx.x * rt, r1 = min(rows, r0 + rt);
  int lo = own ? r0 : INT_MAX, hi = own ? r1 - 1 : -1;
  for (int k = ptr[r0] + (int)threadIdx.x, e = ptr[r1]; k < e; k += blockDim.x) {
    const int c = idx[k];
    lo = min(lo, c);
    hi = max(hi, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ int slo[32], shi[32];
  if ((threadIdx.x & 31) == 0) {
    slo[threadIdx.x >> 5] = lo;
    shi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = min(lo, slo[w]);
      hi = max(hi, shi[w]);
    }
    win[blockIdx.x] = make_int2(lo, hi);
  }
}

// Plan the ring path of M into `win` (device, win_groups(M) entries): true
// when every group's window, and the next group's new columns, fit the ring.
// rows per group: AQP_RING_RT=512 selects the two-CTAs-per-SM form
static int ring_rt() {
  const char *e = getenv("AQP_RING_RT");
  return e && atoi(e) == kRingRT2 ? kRingRT2 : kRingRT;
}
static int win_groups(const DevCsr &M) { return (M.rows + ring_rt() - 1) / ring_rt(); }
static int plan_ring(aqp_ctx *ctx, DevCsr &M, int2 *win, bool &ok) {
  ok = false;
  const int rt = ring_rt(), S = ring_cols(rt), ng = win_groups(M);
  if (ng < 2 * ctx->sm_count) return AQP_OK;  // a strip per SM needs a few groups
  cudaStream_t st = ctx->stream;
  k_win_range<<<ng, 256, 0, st>>>(M.ptr, M.idx, M.rows, rt, M.diag != nullptr, win);
  AQP_CUDA(cudaGetLastError());
  std::vector<int2> h(ng);
  AQP_CUDA(cudaMemcpyAsync(h.data(), win, (size_t)ng * sizeof(int2), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  // monotone windows: prefix maximum of the upper ends, suffix minimum of
  // the lower ends (a group may then only ever need columns the ring adds
  // in order); an empty window sits just above its upper end
  for (int g = 1; g < ng; ++g) h[g].y = std::max(h[g].y, h[g - 1].y);
  for (int g = ng - 2; g >= 0; --g) h[g].x = std::min(h[g].x, h[g + 1].x);
  for (int g = 0; g < ng; ++g)
    if (h[g].x > h[g].y) h[g].x = h[g].y + 1;
  for (int g = 0; g + 1 < ng; ++g) {
    if ((int64_t)h[g + 1].y - h[g].x >= S) return AQP_OK;       // window + next columns exceed the ring
    if ((int64_t)h[g + 1].y - h[g].y > 2 * rt) return AQP_OK;   // two new columns per thread and group
  }
  AQP_CUDA(cudaMemcpyAsync(win, h.data(), (size_t)ng * sizeof(int2), cudaMemcpyHostToDevice, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  ok = true;
  return AQP_OK;
}

// The SELL-32 arrays live in a caller-provided buffer (aqp_problem_attach_sell),
// the offsets in the problem's persistent workspace: dropping them frees nothing.
void free_sell(DevCsr &M, cudaStream_t st) {
  (void)st;
  M.sell_off = nullptr;
  M.sell_idx = nullptr;
  M.sell_val = nullptr;
  M.sell_len = nullptr;
  M.win = nullptr;
  M.win_groups = 0;
  M.win_rt = 0;
  M.win_grid = 0;
  M.sell_perm = nullptr;
}

// 32 * (longest row of each 32-row slice); w[nsl] = 0 so the exclusive scan
// ends with the total
__global__ void k_sell_width(const int *__restrict__ ptr, int rows, int64_t nsl, int64_t *__restrict__ w, bool pair) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nsl) return;
  int mx = 0;
  for (int64_t r = 32 * s; r < 32 * s + 32 && r < rows; ++r) mx = max(mx, ptr[r + 1] - ptr[r]);
  w[s] = sell_width(mx, pair);
}

// SELL-P: sort every 256-row block's rows by length, descending and stable
// (long rows, > kThreadRowMax, and the padding rows of the last block get key
// 0 and sort last); perm[p] = local row at position p; w[slice] = 32 * the
// slice's first (= longest) key; *long_nnz += nonzeros of the long rows.
__global__ void __launch_bounds__(256) k_sellp_sort(const int *__restrict__ ptr, int rows, uint8_t *__restrict__ perm,
                                                    int64_t *__restrict__ w, unsigned long long *long_nnz, bool pair) {
  using Sort = cub::BlockRadixSort<int, 256, 1, int>;
  __shared__ typename Sort::TempStorage tmp;
  const int r = blockIdx.x * 256 + threadIdx.x;
  const int len = r < rows ? ptr[r + 1] - ptr[r] : 0;
  if (len > kThreadRowMax) atomicAdd(long_nnz, (unsigned long long)len);
  int key[1] = {len <= kThreadRowMax ? len : 0};
  int val[1] = {(int)threadIdx.x};
  Sort(tmp).SortDescending(key, val, 0, 6);
  const int64_t p = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (p < rows) perm[p] = (uint8_t)val[0];
  if ((threadIdx.x & 31) == 0) w[p >> 5] = sell_width(key[0], pair);
}

// SELL layout of a non-strict matrix into `off` (+ `perm` for SELL-P):
//   natural SELL-32 when the matrix is uniform and its slices pad <= 1/8
//     (measured on C2: SELL speeds the A pass, 8 nonzeros every row: 38.7 ->
//     33.8 us, but slows the ~2x padded A' and Q passes: 33.0 -> 39.6 and
//     49.0 -> 51.1 us; on C5 A x 2.57 -> 2.07 ms, Q x 1.25 -> 1.17 ms);
//   else, for a matrix that would STAGE (mean row >= 8, A' only: the C5
//     A'), SELL-P (sorted within 256-row blocks) when that pads <= 30% and
//     the long rows hold <= 5% of the nonzeros (C5 P1: 2.55 -> 2.38 ms; on
//     C2's short random rows the block barrier made it slower, 34 -> 44 us);
//   else none (*total = 0).
static int plan_sell(aqp_ctx *ctx, const DevCsr &M, int64_t *off, uint8_t *perm, bool may_sort, bool pair,
                     Bump &scratch, int64_t *total, bool *sorted) {
  *total = 0;
  *sorted = false;
  const char *e = getenv("AQP_SELL");
  if ((e && e[0] == '0') || M.rows == 0 || M.nnz == 0 || !off) return AQP_OK;
  cudaStream_t st = ctx->stream;
  const int64_t nblk = ((int64_t)M.rows + 255) / 256;
  const int64_t nw = nblk * 8;  // slice slots (the last block's beyond-rows slices have width 0)
  scratch.used = 0;
  int64_t *w = (int64_t *)scratch.take((nw + 1) * sizeof(int64_t));
  unsigned long long *lnnz = (unsigned long long *)scratch.take(sizeof(unsigned long long));
  size_t need = 0;
  AQP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, w, off, (int)(nw + 1), st));
  void *tmp = scratch.take(need);
  if (scratch.overflow) return AQP_OK;  // no room to plan: the CSR path serves
  double pad = 0.125;  // AQP_SELL_PAD: A/B knob for the accepted natural padding
  if (const char *pe = getenv("AQP_SELL_PAD")) pad = atof(pe);
  double pad_p = 0.30;  // AQP_SELLP_PAD: the same for SELL-P (0: off)
  if (const char *pe = getenv("AQP_SELLP_PAD")) pad_p = atof(pe);
  int64_t tot = 0;
  if (M.uniform) {
    AQP_CUDA(cudaMemsetAsync(w, 0, (nw + 1) * sizeof(int64_t), st));
    k_sell_width<<<(int)((nw + 256) / 256), 256, 0, st>>>(M.ptr, M.rows, (M.rows + 31) / 32, w, pair);
    AQP_CUDA(cudaGetLastError());
    AQP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, w, off, (int)(nw + 1), st));
    AQP_CUDA(cudaMemcpyAsync(&tot, off + nw, sizeof(tot), cudaMemcpyDeviceToHost, st));
    AQP_CUDA(cudaStreamSynchronize(st));
    if ((double)tot <= (double)M.nnz * (1.0 + pad) + 32) {
      *total = tot;
      return AQP_OK;
    }
  }
  if (!perm || pad_p <= 0.0 || !may_sort || (double)M.nnz < 8.0 * (double)M.rows) return AQP_OK;
  AQP_CUDA(cudaMemsetAsync(w, 0, (nw + 1) * sizeof(int64_t), st));
  AQP_CUDA(cudaMemsetAsync(lnnz, 0, sizeof(unsigned long long), st));
  k_sellp_sort<<<(unsigned)nblk, 256, 0, st>>>(M.ptr, M.rows, perm, w, lnnz, pair);
  AQP_CUDA(cudaGetLastError());
  AQP_CUDA(cub::DeviceScan::ExclusiveSum(tmp, need, w, off, (int)(nw + 1), st));
  unsigned long long ln = 0;
  AQP_CUDA(cudaMemcpyAsync(&tot, off + nw, sizeof(tot), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaMemcpyAsync(&ln, lnnz, sizeof(ln), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  const double short_nnz = (double)M.nnz - (double)ln;
  if ((double)ln <= 0.05 * (double)M.nnz && (double)tot <= short_nnz * (1.0 + pad_p) + 32) {
    *total = tot;
    *sorted = true;
  }
  return AQP_OK;
}

__global__ void k_fill_sellp(const int *__restrict__ ptr, const int *__restrict__ idx, const double *__restrict__ val,
                             int rows, const uint8_t *__restrict__ perm, const int64_t *__restrict__ off, int *sidx,
                             double *sval, bool pair, uint8_t *lens) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= rows) return;
  const int64_t r = (p & ~(int64_t)255) + perm[p];
  const int b = ptr[r], e = ptr[r + 1];
  lens[p] = (uint8_t)min(e - b, 255);  // DevCsr::sell_len (> kThreadRowMax: a long row)
  if (e - b > kThreadRowMax) return;  // long rows stay in the CSR
  const int64_t off0 = off[p >> 5];
  const int lane = (int)(p & 31);
  for (int k = 0; k < e - b; ++k) {
    sidx[sell_pos(off0, lane, k, pair)] = idx[b + k];
    sval[sell_pos(off0, lane, k, pair)] = val[b + k];
  }
}

// ---------------------------------------------------------------- diagonal split (DevCsr::diag)
// (global column of local row r's diagonal = r + row_off: a row shard's Q)
__global__ void k_diag_pos(const int *__restrict__ ptr, const int *__restrict__ idx, int rows, int row_off,
                           int *missing) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  bool found = false;
  for (int k = ptr[r]; k < ptr[r + 1]; ++k) found |= idx[k] == r + row_off;
  if (!found) atomicAdd(missing, 1);
}
// row r loses exactly its diagonal entry: new ptr = old ptr - r
__global__ void k_split_diag(const int *__restrict__ optr, const int *__restrict__ oidx,
                             const double *__restrict__ oval, int rows, int row_off, int *nptr, int *nidx,
                             double *nval, double *diag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > rows) return;
  nptr[r] = optr[r] - r;
  if (r == rows) return;
  int w = optr[r] - r;
  for (int k = optr[r]; k < optr[r + 1]; ++k) {
    if (oidx[k] == r + row_off) {
      diag[r] = oval[k];
    } else {
      nidx[w] = oidx[k];
      nval[w] = oval[k];
      ++w;
    }
  }
}

__global__ void k_row_maxlen(const int *__restrict__ ptr, int rows, int *out) {
  int mx = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    mx = max(mx, ptr[r + 1] - ptr[r]);
  atomicMax(out, mx);
}

// the uniform plan: THREAD items over rows [256 b, 256 b + 256)
__global__ void k_uniform_plan(const int *__restrict__ ptr, int rows, int nitems, PlanItem *plan) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nitems) return;
  PlanItem it{};
  it.row0 = b * kThreads;
  it.row1 = min(rows, (b + 1) * kThreads);
  it.k0 = ptr[it.row0];
  it.k1 = ptr[it.row1];
  it.kind = kItemThread;
  plan[b] = it;
}

// Plan the SpMV work of M (rows from M.ptr on the device, or from the given
// host copy).  Without a host copy, a uniform matrix (every row <= the
// THREAD length, no staging, not strict -- the common case, every C2 / C5
// pass but A') is planned on the device; otherwise the row pointers come to
// the host for plan_rows.
int finish_plan(aqp_ctx *ctx, DevCsr &M, const int *host_ptr32, const int64_t *host_ptr64, bool strict,
                PlanItem *plan_dev, int64_t plan_cap, double *seg_part, unsigned *seg_ticket,
                int64_t seg_cap, bool may_stage) {
  int nlong = 0;
  // STAGED items for matrices with long-enough rows (see kItemStaged)
  // measured on C5 (n = m = 5e7, 10 nnz / row): STAGED speeds the A' pass
  // (P1, 2.80 -> 2.55 ms) but slows the A pass (P2, whose epilogue operands
  // are held across the staging barrier: 2.51 -> 2.86 ms), so only A' stages
  double staged_min = may_stage ? 8.0 : 1e300;
  if (const char *e = getenv("AQP_STAGED_MIN"))  // A/B knob for the matrices that may stage (A')
    if (may_stage) staged_min = atof(e);
  cudaStream_t st = ctx->stream;
  free_sell(M, st);  // a re-plan drops the SELL copy (aqp_problem_attach_sell rebuilds it)
  std::vector<int> dev_ptr_copy;
  if (!host_ptr32 && !host_ptr64) {
    const bool staged = !strict && M.rows > 0 && (double)M.nnz >= staged_min * (double)M.rows;
    if (!strict && !staged && M.rows > 0) {
      int *dmax = (int *)seg_ticket;  // seg_ticket is zeroed scratch until the plan is in place
      int mx = 0;
      AQP_CUDA(cudaMemsetAsync(dmax, 0, sizeof(int), st));
      k_row_maxlen<<<std::min(148 * 16, (M.rows + 255) / 256), 256, 0, st>>>(M.ptr, M.rows, dmax);
      AQP_CUDA(cudaGetLastError());
      AQP_CUDA(cudaMemcpyAsync(&mx, dmax, sizeof(int), cudaMemcpyDeviceToHost, st));
      AQP_CUDA(cudaMemsetAsync(dmax, 0, sizeof(int), st));
      AQP_CUDA(cudaStreamSynchronize(st));
      if (mx <= kThreadRowMax) {
        const int nitems = (M.rows + kThreads - 1) / kThreads;
        if (nitems > plan_cap) return fail(AQP_ENOMEM, "plan capacity exceeded");
        k_uniform_plan<<<(nitems + 255) / 256, 256, 0, st>>>(M.ptr, M.rows, nitems, plan_dev);
        AQP_CUDA(cudaGetLastError());
        M.plan = plan_dev;
        M.nitems = nitems;
        M.smem_bytes = 0;
        M.uniform = 1;
        M.nlongseg = 0;
        M.seg_part = seg_part;
        M.seg_ticket = seg_ticket;
        step_mark(st, "  finish_plan.device_uniform");
        return AQP_OK;
      }
    }
    dev_ptr_copy.resize((size_t)M.rows + 1);
    AQP_CUDA(cudaMemcpyAsync(dev_ptr_copy.data(), M.ptr, (M.rows + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
    AQP_CUDA(cudaStreamSynchronize(st));
    host_ptr32 = dev_ptr_copy.data();
  }
  const int64_t nnz_rows = M.rows > 0 ? (host_ptr64 ? host_ptr64[M.rows] - host_ptr64[0]
                                                    : (int64_t)host_ptr32[M.rows] - host_ptr32[0]) : 0;
  const bool staged = !strict && M.rows > 0 && (double)nnz_rows >= staged_min * (double)M.rows;
  std::vector<PlanItem> items = host_ptr64 ? plan_rows(host_ptr64, M.rows, strict, &nlong, staged)
                                           : plan_rows(host_ptr32, M.rows, strict, &nlong, staged);
  step_mark(ctx->stream, "  finish_plan.plan_rows");
  if ((int64_t)items.size() > plan_cap) return fail(AQP_ENOMEM, "plan capacity exceeded");
  if (nlong > seg_cap) return fail(AQP_ENOMEM, "segment capacity exceeded");
  AQP_CUDA(cudaMemcpyAsync(plan_dev, items.data(), items.size() * sizeof(PlanItem), cudaMemcpyHostToDevice,
                           ctx->stream));
  AQP_CUDA(cudaStreamSynchronize(ctx->stream));  // `items` is pageable and local
  M.plan = plan_dev;
  M.nitems = (int)items.size();
  bool warp_items = false;
  for (const PlanItem &it : items) warp_items |= it.kind == kItemWarp || it.kind == kItemStaged;
  M.smem_bytes = warp_items ? kTileNnz * (int)(sizeof(double) + sizeof(int)) : 0;
  // uniform plans let the kernel derive its rows from blockIdx (no plan load)
  bool uniform = M.rows > 0;
  for (size_t b = 0; b < items.size() && uniform; ++b)
    uniform = items[b].kind == kItemThread && items[b].row0 == (int)(b * kThreads) &&
              items[b].row1 == (int)std::min<int64_t>((int64_t)(b + 1) * kThreads, M.rows);
  M.uniform = uniform ? 1 : 0;
  M.nlongseg = nlong;
  M.seg_part = seg_part;
  M.seg_ticket = seg_ticket;
  return AQP_OK;
}

// The CSR plan of a deferred A' (see aqp_problem::at_plan_deferred): run when
// a solver is created without the SELL-P copy attached (or SELL-P was not
// chosen); the SELL-P attach replaces the plan by its own (one block per 256
// rows), so the planning pass is skipped altogether on the common path.
int plan_deferred_at(aqp_problem *p) {
  if (!p->at_plan_deferred) return AQP_OK;
  CsrStore &t = p->sAt;
  AQP_TRY(finish_plan(p->ctx, p->At, nullptr, nullptr, false, t.plan, t.plan_cap, t.seg_part, t.seg_ticket,
                      t.seg_cap, true));
  p->at_plan_deferred = false;
  p->info.at_items = p->At.nitems;
  return AQP_OK;
}

// Persistent storage of one device CSR with its plan.
void layout_csr(Bump &b, CsrStore &s, int64_t rows, int64_t nnz) {
  s.ptr = (int *)b.take((rows + 1) * sizeof(int));
  s.idx = (int *)b.take(std::max<int64_t>(nnz, 1) * sizeof(int));
  s.val = (double *)b.take(std::max<int64_t>(nnz, 1) * sizeof(double));
  s.cap_nnz = nnz;
  s.plan_cap = plan_capacity(rows, nnz);
  s.plan = (PlanItem *)b.take(s.plan_cap * sizeof(PlanItem));
  s.seg_cap = nnz / kSegNnz + nnz / kTileNnz + 2;  // each long row adds at most one partial segment
  s.seg_part = (double *)b.take(2 * s.seg_cap * sizeof(double));
  s.seg_ticket = (unsigned *)b.take(s.seg_cap * sizeof(unsigned));
  s.sell_off = (int64_t *)b.take(((rows + 255) / 256 * 8 + 2) * sizeof(int64_t));
  s.sell_perm = (uint8_t *)b.take(std::max<int64_t>(rows, 1));
}

// Upload an int64 CSR (device pointers) into int32 storage and plan it.
int upload_csr(aqp_ctx *ctx, CsrStore &s, DevCsr &M, int64_t rows, int64_t cols, const int64_t *d_ptr,
               const int64_t *d_idx, const double *d_val, int64_t nnz, const int64_t *host_ptr, bool strict,
               int *d_bad) {
  cudaStream_t st = ctx->stream;
  AQP_TRY(to_i32(d_ptr, s.ptr, rows + 1, INT32_MAX, d_bad, st));
  AQP_TRY(to_i32(d_idx, s.idx, nnz, cols - 1, d_bad, st));
  if (nnz) AQP_CUDA(cudaMemcpyAsync(s.val, d_val, nnz * sizeof(double), cudaMemcpyDeviceToDevice, st));
  AQP_CUDA(cudaMemsetAsync(s.seg_ticket, 0, s.seg_cap * sizeof(unsigned), st));
  step_mark(st, "  upload_csr.convert");
  M.rows = (int)rows;
  M.cols = (int)cols;
  M.nnz = nnz;
  M.ptr = s.ptr;
  M.idx = s.idx;
  M.val = s.val;
  // non-strict plans start on the device (uniform matrices never visit the host)
  return finish_plan(ctx, M, nullptr, strict ? host_ptr : nullptr, strict, s.plan, s.plan_cap, s.seg_part, s.seg_ticket, s.seg_cap,
                     false);
}

// Transpose of an uploaded CSR (src) into storage t, restricted to the
// source columns [col0, col1) (default: all): output row i is source column
// col0 + i, its column indices are source rows + row_base (the global row of
// the source's row 0; a row shard's A block), ascending -- a STABLE sort, so
// the row-sequential product equals the Cython scatter order.  out_cols is
// the output's column count (default: src.rows).
// Scratch: rid(nnz) keys(nnz) keys2(nnz) vals(nnz) vals2(nnz) counts(rows_t+1) + cub.
int transpose_csr(aqp_ctx *ctx, const DevCsr &src, CsrStore &t, DevCsr &T, bool strict, Bump &scratch, int64_t col0,
                  int64_t col1, int64_t row_base, int64_t out_cols, bool *deferred) {
  cudaStream_t st = ctx->stream;
  const int64_t nnz = src.nnz;
  if (col1 < 0) col1 = src.cols;
  if (out_cols < 0) out_cols = src.rows;
  const int rows_t = (int)(col1 - col0);
  const bool window = col0 != 0 || col1 != src.cols;
  scratch.used = 0;
  int *rid = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  int *keys = window ? (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4) : nullptr;
  int *keys2 = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  int *vals = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  int *vals2 = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  int *counts = (int *)scratch.take((int64_t)(rows_t + 2) * 4);
  size_t tb = sort_temp_bytes(std::max<int64_t>(nnz, rows_t + 2));
  void *tmp = scratch.take(tb);
  if (scratch.overflow) return fail(AQP_ENOMEM, "transpose scratch too small");
  AQP_CUDA(cudaMemsetAsync(counts, 0, (rows_t + 2) * sizeof(int), st));
  int64_t nnz_t = nnz;
  if (nnz) {
    const int *sort_keys = src.idx;
    if (window) {
      k_tkeys<<<setup_grid(nnz), 256, 0, st>>>(src.idx, nnz, (int)col0, (int)col1, keys);
      sort_keys = keys;
    }
    k_row_ids<<<setup_grid(src.rows), 256, 0, st>>>(src.ptr, src.rows, rid);
    k_iota<<<setup_grid(nnz), 256, 0, st>>>(vals, nnz);
    AQP_CUDA(cudaGetLastError());
    int end_bit = 1;
    while ((1LL << end_bit) <= (int64_t)rows_t) ++end_bit;
    size_t need = tb;
    AQP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, sort_keys, keys2, vals, vals2, (int)nnz, 0, end_bit, st));
    k_run_counts<<<setup_grid(nnz), 256, 0, st>>>(keys2, nnz, counts);  // counts[rows_t]: outside the window
    AQP_CUDA(cudaGetLastError());
    if (window) {
      int outside = 0;
      AQP_CUDA(cudaMemcpyAsync(&outside, counts + rows_t, sizeof(int), cudaMemcpyDeviceToHost, st));
      AQP_CUDA(cudaStreamSynchronize(st));
      nnz_t = nnz - outside;
      AQP_CUDA(cudaMemsetAsync(counts + rows_t, 0, sizeof(int), st));
    }
    if (nnz_t > t.cap_nnz) return fail(AQP_ENOMEM, "transpose: more nonzeros than the storage holds");
    k_gather_t<<<setup_grid(nnz_t), 256, 0, st>>>(vals2, rid, src.val, nnz_t, (int)row_base, t.idx, t.val);
    AQP_CUDA(cudaGetLastError());
  }
  AQP_TRY(counts_to_ptr(counts, rows_t, t.ptr, tmp, tb, st));
  AQP_CUDA(cudaMemsetAsync(t.seg_ticket, 0, t.seg_cap * sizeof(unsigned), st));
  T.rows = rows_t;
  T.cols = (int)out_cols;
  T.nnz = nnz_t;
  T.ptr = t.ptr;
  T.idx = t.idx;
  T.val = t.val;
  if (deferred) {
    // a staged A' (mean row >= the staging threshold: its plan is never
    // uniform, so SELL planning does not depend on it) waits for
    // plan_deferred_at; everything else is planned now
    double staged_min = 8.0;
    if (const char *e = getenv("AQP_STAGED_MIN")) staged_min = atof(e);
    *deferred = !strict && T.rows > 0 && (double)T.nnz >= staged_min * (double)T.rows;
    if (*deferred) {
      free_sell(T, st);
      T.plan = nullptr;
      T.nitems = 0;
      T.uniform = 0;
      T.smem_bytes = 0;
      T.nlongseg = 0;
      T.seg_part = t.seg_part;
      T.seg_ticket = t.seg_ticket;
      return AQP_OK;
    }
  }
  return finish_plan(ctx, T, nullptr, nullptr, strict, t.plan, t.plan_cap, t.seg_part, t.seg_ticket, t.seg_cap,
                     true);
}

// Full symmetric expansion of an uploaded upper-triangle CSR U whose row 0 is
// global row row_base (a row shard's P block; 0 for a whole n x n triangle),
// restricted to the output rows [r0, r1) (default: all of U's rows).  Each
// output row is [mirrored lower part | stored upper part], both ascending, in
// global column indices.
int symmetrize_csr(aqp_ctx *ctx, const DevCsr &U, CsrStore &f, DevCsr &F, bool strict, Bump &scratch,
                   int64_t *nfull_out, int64_t row_base, int64_t r0, int64_t r1) {
  cudaStream_t st = ctx->stream;
  const int64_t nnz = U.nnz;
  if (r1 < 0) r1 = U.rows;
  const int n = (int)(r1 - r0);  // output rows
  const int64_t n2 = 2 * nnz;
  scratch.used = 0;
  int *rid = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  int *keys = (int *)scratch.take(std::max<int64_t>(n2, 1) * 4);
  int *keys2 = (int *)scratch.take(std::max<int64_t>(n2, 1) * 4);
  int *vals = (int *)scratch.take(std::max<int64_t>(n2, 1) * 4);
  int *vals2 = (int *)scratch.take(std::max<int64_t>(n2, 1) * 4);
  int *counts = (int *)scratch.take((int64_t)(n + 2) * 4);
  size_t tb = sort_temp_bytes(std::max<int64_t>(n2, n + 2));
  void *tmp = scratch.take(tb);
  if (scratch.overflow) return fail(AQP_ENOMEM, "symmetrize scratch too small");
  AQP_CUDA(cudaMemsetAsync(counts, 0, (n + 2) * sizeof(int), st));
  int64_t nfull = 0;
  if (nnz) {
    k_row_ids<<<setup_grid(U.rows), 256, 0, st>>>(U.ptr, U.rows, rid);
    k_sym_keys<<<setup_grid(nnz), 256, 0, st>>>(rid, U.idx, nnz, (int)row_base, (int)r0, (int)r1, keys);
    k_iota<<<setup_grid(n2), 256, 0, st>>>(vals, n2);
    AQP_CUDA(cudaGetLastError());
    int end_bit = 1;
    while ((1LL << end_bit) <= (int64_t)n) ++end_bit;
    size_t need = tb;
    step_mark(st, "  symmetrize.keys");
    AQP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, need, keys, keys2, vals, vals2, (int)n2, 0, end_bit, st));
    k_run_counts<<<setup_grid(n2), 256, 0, st>>>(keys2, n2, counts);  // counts[n] = #sentinels (diagonal mirrors, outside)
    AQP_CUDA(cudaGetLastError());
    step_mark(st, "  symmetrize.sort");
    int ndiag = 0;
    AQP_CUDA(cudaMemcpyAsync(&ndiag, counts + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    AQP_CUDA(cudaStreamSynchronize(st));
    nfull = n2 - ndiag;
    if (nfull > f.cap_nnz) return fail(AQP_ENOMEM, "symmetrize: more nonzeros than the storage holds");
    k_sym_gather<<<setup_grid(nfull), 256, 0, st>>>(vals2, rid, U.idx, U.val, nnz, nfull, (int)row_base, f.idx,
                                                    f.val);
    AQP_CUDA(cudaGetLastError());
  }
  AQP_CUDA(cudaMemsetAsync(counts + n, 0, sizeof(int), st));
  AQP_TRY(counts_to_ptr(counts, n, f.ptr, tmp, tb, st));
  AQP_CUDA(cudaMemsetAsync(f.seg_ticket, 0, f.seg_cap * sizeof(unsigned), st));
  F.rows = n;
  F.cols = U.cols;
  F.nnz = nfull;
  F.row_off = (int)r0;
  F.ptr = f.ptr;
  F.idx = f.idx;
  F.val = f.val;
  *nfull_out = nfull;
  step_mark(st, "  symmetrize.gather_scan");
  return finish_plan(ctx, F, nullptr, nullptr, strict, f.plan, f.plan_cap, f.seg_part, f.seg_ticket, f.seg_cap,
                     false);
}

size_t transpose_scratch_bytes(int64_t nnz, int64_t cols) {
  Bump b;
  for (int i = 0; i < 5; ++i) b.take(std::max<int64_t>(nnz, 1) * 4);
  b.take((cols + 2) * 4);
  b.take(sort_temp_bytes(std::max<int64_t>(nnz, cols + 2)));
  return b.used + 256;
}

size_t symmetrize_scratch_bytes(int64_t nnz, int64_t n) {
  Bump b;
  b.take(std::max<int64_t>(nnz, 1) * 4);
  for (int i = 0; i < 4; ++i) b.take(std::max<int64_t>(2 * nnz, 1) * 4);
  b.take((n + 2) * 4);
  b.take(sort_temp_bytes(std::max<int64_t>(2 * nnz, n + 2)));
  return b.used + 256;
}

int build_cones(aqp_ctx *ctx, const double *lo, const double *hi, int64_t n, int8_t *dual, int8_t *recc,
                int is_y) {
  if (n == 0) return AQP_OK;
  k_cones<<<setup_grid(n), 256, 0, ctx->stream>>>(lo, hi, n, dual, recc, is_y);
  AQP_CUDA(cudaGetLastError());
  return AQP_OK;
}

}  // namespace aqp

using namespace aqp;

// ====================================================================== C ABI
extern "C" {

int aqp_abi_version(void) { return AQP_ABI_VERSION; }
const char *aqp_last_error(void) { return g_last_error.c_str(); }

int aqp_ctx_create(int device, void *stream, aqp_ctx **out) {
  if (!out) return fail(AQP_EINVAL, "out is NULL");
  AQP_CUDA(cudaSetDevice(device));
  aqp_ctx *c = new aqp_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  const int rc = xfer_init(device);  // the staged-copy pool (aqp_xfer.cu), once per process
  if (rc != AQP_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return AQP_OK;
}

int aqp_ctx_destroy(aqp_ctx *ctx) {
  if (ctx && ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx && ctx->bounce) cudaFreeHost(ctx->bounce);
  delete ctx;
  return AQP_OK;
}

static int check_desc(const aqp_problem_desc *d) {
  if (!d) return fail(AQP_EINVAL, "desc is NULL");
  if (d->n < 0 || d->m < 0) return fail(AQP_EINVAL, "negative dimension");
  if (d->n >= INT32_MAX || d->m >= INT32_MAX || d->a_nnz >= INT32_MAX / 2 || d->q_nnz >= INT32_MAX / 4 ||
      d->r_nnz >= INT32_MAX / 2 || d->r_rows >= INT32_MAX)
    return fail(AQP_ERANGE, "instance exceeds int32 device indexing");
  if (d->quad_kind < AQP_QUAD_DIAGONAL || d->quad_kind > AQP_QUAD_SPARSE_LOW_RANK)
    return fail(AQP_EINVAL, "unknown quad kind");
  return AQP_OK;
}

// Move the diagonal of a uniform-plan full symmetric Q out of the CSR (every
// row must hold one); scratch holds the old arrays during the compaction.
static int split_q_diag(aqp_ctx *ctx, aqp_problem *p, Bump &scratch) {
  DevCsr &M = p->Q;
  const char *e = getenv("AQP_SPLIT_DIAG");
  if ((e && e[0] == '0') || !M.uniform || M.rows == 0) return AQP_OK;
  cudaStream_t st = ctx->stream;
  const int n = M.rows;
  const int64_t nnz = M.nnz;
  scratch.used = 0;
  int *missing = (int *)scratch.take(64);
  int *oidx = (int *)scratch.take(std::max<int64_t>(nnz, 1) * 4);
  double *oval = (double *)scratch.take(std::max<int64_t>(nnz, 1) * 8);
  int *optr = (int *)scratch.take((int64_t)(n + 1) * 4);
  if (scratch.overflow) return AQP_OK;  // not enough scratch: keep the diagonal in the CSR
  AQP_CUDA(cudaMemsetAsync(missing, 0, 4, st));
  k_diag_pos<<<(n + 255) / 256, 256, 0, st>>>(M.ptr, M.idx, n, M.row_off, missing);
  AQP_CUDA(cudaGetLastError());
  int miss = 0;
  AQP_CUDA(cudaMemcpyAsync(&miss, missing, 4, cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  if (miss) return AQP_OK;
  CsrStore &s = p->sQ;
  AQP_CUDA(cudaMemcpyAsync(oidx, M.idx, nnz * 4, cudaMemcpyDeviceToDevice, st));
  AQP_CUDA(cudaMemcpyAsync(oval, M.val, nnz * 8, cudaMemcpyDeviceToDevice, st));
  AQP_CUDA(cudaMemcpyAsync(optr, M.ptr, (int64_t)(n + 1) * 4, cudaMemcpyDeviceToDevice, st));
  k_split_diag<<<(n + 256) / 256, 256, 0, st>>>(optr, oidx, oval, n, M.row_off, s.ptr, s.idx, s.val, p->qdiag);
  AQP_CUDA(cudaGetLastError());
  M.nnz = nnz - n;
  M.diag = p->qdiag;
  M.ptr = s.ptr;
  AQP_TRY(finish_plan(ctx, M, nullptr, nullptr, false, s.plan, s.plan_cap, s.seg_part, s.seg_ticket, s.seg_cap,
                      false));
  if (!M.uniform) return fail(AQP_ECUDA, "diagonal split changed the Q plan kind");
  return AQP_OK;
}

// persistent sizes: the whole problem, or (shard) this rank's rows only
struct ProbDims {
  int64_t nl, ml;        // local rows (x side, y side)
  int64_t a_nnz, at_nnz;  // nonzeros stored for A and A'
  int64_t q_nnz;         // capacity of the full symmetric Q rows
  int64_t r_nnz;         // nonzeros of the (local) R
};
static ProbDims dims_of(const aqp_problem_desc *d) {
  const aqp_shard_desc *sh = d->shard;
  ProbDims g;
  if (!sh) {
    g.nl = d->n;
    g.ml = d->m;
    g.a_nnz = g.at_nnz = d->a_nnz;
    g.q_nnz = 2 * d->q_nnz;
  } else {
    g.nl = sh->n1 - sh->n0;
    g.ml = sh->m1 - sh->m0;
    g.a_nnz = sh->a_local_nnz;
    g.at_nnz = sh->at_local_nnz;
    g.q_nnz = sh->q_local_nnz;
  }
  g.r_nnz = d->r_nnz;
  return g;
}

static void layout_problem(Bump &b, const aqp_problem_desc *d, aqp_problem *p) {
  const ProbDims g = dims_of(d);
  const int64_t n = g.nl, m = g.ml;
  layout_csr(b, p->sA, m, g.a_nnz);
  layout_csr(b, p->sAt, n, g.at_nnz);
  if (d->quad_kind != AQP_QUAD_DIAGONAL) {
    layout_csr(b, p->sQ, n, g.q_nnz);
    p->qdiag = (double *)b.take(std::max<int64_t>(n, 1) * 8);
  }
  if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK) {
    if (d->r_dense) {
      p->sR.val = (double *)b.take(std::max<int64_t>(d->r_rows * n, 1) * 8);
    } else {
      layout_csr(b, p->sR, d->r_rows, g.r_nnz);
      layout_csr(b, p->sRt, n, g.r_nnz);
    }
  }
  p->c = (double *)b.take(std::max<int64_t>(n, 1) * 8);
  p->vlo = (double *)b.take(std::max<int64_t>(n, 1) * 8);
  p->vhi = (double *)b.take(std::max<int64_t>(n, 1) * 8);
  p->qd = (double *)b.take(std::max<int64_t>(n, 1) * 8);
  p->clo = (double *)b.take(std::max<int64_t>(m, 1) * 8);
  p->chi = (double *)b.take(std::max<int64_t>(m, 1) * 8);
  p->cone_r = (int8_t *)b.take(std::max<int64_t>(n, 1));
  p->recc_x = (int8_t *)b.take(std::max<int64_t>(n, 1));
  p->cone_y = (int8_t *)b.take(std::max<int64_t>(m, 1));
  p->recc_s = (int8_t *)b.take(std::max<int64_t>(m, 1));
  p->bad = (int *)b.take(64);
  p->setup_scratch = b.take(256);
}

static int check_shard(const aqp_problem_desc *d) {
  const aqp_shard_desc *sh = d->shard;
  if (!sh) return AQP_OK;
  if (sh->nranks < 1 || sh->nranks > kMaxRanks || sh->rank < 0 || sh->rank >= sh->nranks)
    return fail(AQP_EINVAL, "rank / nranks out of range (at most 8 ranks)");
  if (sh->n0 < 0 || sh->n1 > d->n || sh->n0 >= sh->n1 || sh->m0 < 0 || sh->m1 > d->m || sh->m0 >= sh->m1)
    return fail(AQP_EINVAL, "shard row ranges must be non-empty and inside [0,n) / [0,m)");
  if (sh->a_row0 < 0 || sh->a_rows < 0 || sh->a_row0 + sh->a_rows > d->m || sh->m0 < sh->a_row0 ||
      sh->m1 > sh->a_row0 + sh->a_rows)
    return fail(AQP_EINVAL, "the A block must cover the owned rows [m0,m1)");
  if (d->quad_kind != AQP_QUAD_DIAGONAL && (sh->q_row0 < 0 || sh->q_row0 > sh->n0))
    return fail(AQP_EINVAL, "the P block must start at or before n0");
  if (sh->nl_cap < sh->n1 - sh->n0 || sh->ml_cap < sh->m1 - sh->m0) return fail(AQP_EINVAL, "row capacity too small");
  for (int k = 0; k < sh->nranks; ++k)
    if (sh->xw[2 * k] < 0 || sh->xw[2 * k + 1] > d->n || sh->xw[2 * k] > sh->xw[2 * k + 1] || sh->yw[2 * k] < 0 ||
        sh->yw[2 * k + 1] > d->m || sh->yw[2 * k] > sh->yw[2 * k + 1])
      return fail(AQP_EINVAL, "gather window outside [0,n) / [0,m)");
  const int r = sh->rank;
  if (sh->xw[2 * r] > sh->n0 || sh->xw[2 * r + 1] < sh->n1 || sh->yw[2 * r] > sh->m0 || sh->yw[2 * r + 1] < sh->m1)
    return fail(AQP_EINVAL, "a rank's gather windows must cover its own rows");
  if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK && d->r_rows > kMaxVec)
    return fail(AQP_EINVAL, "row-sharded low-rank Q supports at most 256 factor rows (R x is all-reduced)");
  return AQP_OK;
}

int aqp_problem_sizes(const aqp_problem_desc *d, size_t *persistent_bytes, size_t *scratch_bytes) {
  AQP_TRY(check_desc(d));
  AQP_TRY(check_shard(d));
  aqp_problem tmp;
  Bump b;
  layout_problem(b, d, &tmp);
  const aqp_shard_desc *sh = d->shard;
  const ProbDims g = dims_of(d);
  size_t sc;
  if (!sh) {
    sc = transpose_scratch_bytes(d->a_nnz, d->n);
  } else {
    // the int32 A block sits at the front of the scratch during its transpose
    const size_t blk = (size_t)(sh->a_rows + 1) * 4 + (size_t)std::max<int64_t>(d->a_nnz, 1) * 4 + 1024;
    sc = blk + transpose_scratch_bytes(d->a_nnz, g.nl);
  }
  if (d->quad_kind != AQP_QUAD_DIAGONAL) {
    // the int32 upper triangle (block) sits at the front of the scratch during the expansion
    const int64_t urows = sh ? sh->n1 - sh->q_row0 : d->n;
    const size_t up = (size_t)(urows + 1) * 4 + (size_t)std::max<int64_t>(d->q_nnz, 1) * 12 + 1024;
    sc = std::max(sc, up + symmetrize_scratch_bytes(d->q_nnz, g.nl));
  }
  if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK && !d->r_dense)
    sc = std::max(sc, transpose_scratch_bytes(d->r_nnz, g.nl));
  if (persistent_bytes) *persistent_bytes = b.used + 256;
  if (scratch_bytes) *scratch_bytes = sc;
  return AQP_OK;
}

// A row shard's A: rows [m0,m1) of the uploaded block, and A': the block's
// columns [n0,n1) transposed (column indices = global rows of A).
static int shard_a(aqp_ctx *ctx, aqp_problem *p, const aqp_problem_desc *d, const int64_t *host_ptr, void *scratch,
                   size_t scratch_bytes) {
  const aqp_shard_desc *sh = d->shard;
  cudaStream_t st = ctx->stream;
  Bump ub;
  ub.base = scratch;
  ub.cap = scratch_bytes;
  int *bptr = (int *)ub.take((sh->a_rows + 1) * 4);
  int *bidx = (int *)ub.take(std::max<int64_t>(d->a_nnz, 1) * 4);
  if (ub.overflow) return fail(AQP_ENOMEM, "scratch too small for the A block");
  AQP_TRY(to_i32(d->a_indptr, bptr, sh->a_rows + 1, INT32_MAX, p->bad, st));
  AQP_TRY(to_i32(d->a_indices, bidx, d->a_nnz, d->n - 1, p->bad, st));
  DevCsr B;
  B.rows = (int)sh->a_rows;
  B.cols = (int)d->n;
  B.nnz = d->a_nnz;
  B.ptr = bptr;
  B.idx = bidx;
  B.val = d->a_data;
  // A = rows [m0, m1) of the block, copied (rebased) into its own storage
  const int64_t r0 = sh->m0 - sh->a_row0, rows = sh->m1 - sh->m0;
  const int64_t k0 = host_ptr[r0] - host_ptr[0], k1 = host_ptr[r0 + rows] - host_ptr[0];
  if (k1 - k0 != sh->a_local_nnz) return fail(AQP_EINVAL, "a_local_nnz does not match the A block");
  k_rebase_ptr<<<setup_grid(rows + 1), 256, 0, st>>>(bptr, r0, rows, p->sA.ptr);
  AQP_CUDA(cudaGetLastError());
  if (k1 > k0) {
    AQP_CUDA(cudaMemcpyAsync(p->sA.idx, bidx + k0, (k1 - k0) * 4, cudaMemcpyDeviceToDevice, st));
    AQP_CUDA(cudaMemcpyAsync(p->sA.val, d->a_data + k0, (k1 - k0) * 8, cudaMemcpyDeviceToDevice, st));
  }
  AQP_CUDA(cudaMemsetAsync(p->sA.seg_ticket, 0, p->sA.seg_cap * sizeof(unsigned), st));
  DevCsr &A = p->A;
  A.rows = (int)rows;
  A.cols = (int)d->n;
  A.nnz = k1 - k0;
  A.ptr = p->sA.ptr;
  A.idx = p->sA.idx;
  A.val = p->sA.val;
  std::vector<int64_t> hp((size_t)rows + 1);
  for (int64_t i = 0; i <= rows; ++i) hp[i] = host_ptr[r0 + i] - host_ptr[r0];
  AQP_TRY(finish_plan(ctx, A, nullptr, hp.data(), false, p->sA.plan, p->sA.plan_cap, p->sA.seg_part,
                      p->sA.seg_ticket, p->sA.seg_cap, false));
  Bump rest;
  const size_t used = (ub.used + 255) & ~size_t(255);
  rest.base = static_cast<char *>(scratch) + used;
  rest.cap = scratch_bytes - used;
  AQP_TRY(transpose_csr(ctx, B, p->sAt, p->At, false, rest, sh->n0, sh->n1, sh->a_row0, d->m));
  if (p->At.nnz != sh->at_local_nnz) return fail(AQP_EINVAL, "at_local_nnz does not match the A block");
  return AQP_OK;
}

int aqp_problem_create(aqp_ctx *ctx, const aqp_problem_desc *d, const int64_t *host_a_indptr,
                       const int64_t *host_q_indptr, const int64_t *host_r_indptr, void *persistent,
                       size_t persistent_bytes, void *scratch, size_t scratch_bytes, aqp_problem **out) {
  (void)host_q_indptr;
  AQP_TRY(check_desc(d));
  AQP_TRY(check_shard(d));
  if (!ctx || !out || !persistent || !host_a_indptr) return fail(AQP_EINVAL, "NULL argument");
  if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK && !host_r_indptr) return fail(AQP_EINVAL, "R indptr missing");
  AQP_CUDA(cudaSetDevice(ctx->device));
  const aqp_shard_desc *sh = d->shard;
  const ProbDims g = dims_of(d);
  aqp_problem *p = new aqp_problem();
  p->ctx = ctx;
  p->n = d->n;
  p->m = d->m;
  p->n1 = d->n;
  p->m1 = d->m;
  p->nl_cap = p->xw_cap = d->n;
  p->ml_cap = p->yw_cap = d->m;
  for (int k = 0; k < kMaxRanks; ++k) {
    p->xwin[2 * k + 1] = d->n;
    p->ywin[2 * k + 1] = d->m;
  }
  if (sh) {
    p->rank = sh->rank;
    p->nranks = sh->nranks;
    p->n0 = sh->n0;
    p->n1 = sh->n1;
    p->m0 = sh->m0;
    p->m1 = sh->m1;
    p->nl_cap = sh->nl_cap;
    p->ml_cap = sh->ml_cap;
    p->xw_cap = p->yw_cap = 0;
    for (int k = 0; k < 2 * kMaxRanks; ++k) {
      p->xwin[k] = k < 2 * sh->nranks ? sh->xw[k] : 0;
      p->ywin[k] = k < 2 * sh->nranks ? sh->yw[k] : 0;
    }
    for (int k = 0; k < sh->nranks; ++k) {
      p->xw_cap = std::max(p->xw_cap, sh->xw[2 * k + 1] - sh->xw[2 * k]);
      p->yw_cap = std::max(p->yw_cap, sh->yw[2 * k + 1] - sh->yw[2 * k]);
    }
  }
  p->quad_kind = d->quad_kind;
  Bump b;
  b.base = persistent;
  b.cap = persistent_bytes;
  layout_problem(b, d, p);
  if (b.overflow) {
    delete p;
    return fail(AQP_ENOMEM, "persistent workspace too small");
  }
  Bump sc;
  sc.base = scratch;
  sc.cap = scratch_bytes;
  cudaStream_t st = ctx->stream;
  int rc = AQP_OK;
  auto cleanup = [&](int code) {
    for (DevCsr *M : {&p->A, &p->At, &p->Q, &p->R, &p->Rt}) free_sell(*M, st);
    delete p;
    return code;
  };
  AQP_CUDA(cudaMemsetAsync(p->bad, 0, 64, st));
  StepTimer tm(st);
  if (!sh) {
    rc = upload_csr(ctx, p->sA, p->A, d->m, d->n, d->a_indptr, d->a_indices, d->a_data, d->a_nnz, host_a_indptr,
                    false, p->bad);
    if (rc) return cleanup(rc);
    tm("A_convert_plan");
    rc = transpose_csr(ctx, p->A, p->sAt, p->At, false, sc, 0, -1, 0, -1, &p->at_plan_deferred);
    tm("At_transpose_plan");
  } else {
    rc = shard_a(ctx, p, d, host_a_indptr, scratch, scratch_bytes);
  }
  if (rc) return cleanup(rc);
  p->q_full_nnz = 0;
  const int64_t n = g.nl, m = g.ml;  // local rows
  if (d->quad_kind == AQP_QUAD_DIAGONAL) {
    if (n) AQP_CUDA(cudaMemcpyAsync(p->qd, d->q_values, n * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    // the upper triangle (a shard: its block of rows [q_row0, n1)) is
    // converted to int32 at the front of the scratch, then expanded into
    // the full symmetric rows this problem stores
    const int64_t urow0 = sh ? sh->q_row0 : 0;
    const int64_t urows = sh ? sh->n1 - sh->q_row0 : d->n;
    DevCsr U;
    CsrStore su;
    Bump ub;
    ub.base = scratch;
    ub.cap = scratch_bytes;
    su.ptr = (int *)ub.take((urows + 1) * 4);
    su.idx = (int *)ub.take(std::max<int64_t>(d->q_nnz, 1) * 4);
    su.val = (double *)ub.take(std::max<int64_t>(d->q_nnz, 1) * 8);
    if (ub.overflow) return cleanup(fail(AQP_ENOMEM, "scratch too small for Q upload"));
    rc = to_i32(d->q_indptr, su.ptr, urows + 1, INT32_MAX, p->bad, st);
    if (!rc) rc = to_i32(d->q_indices, su.idx, d->q_nnz, d->n - 1, p->bad, st);
    if (rc) return cleanup(rc);
    if (d->q_nnz) AQP_CUDA(cudaMemcpyAsync(su.val, d->q_data, d->q_nnz * 8, cudaMemcpyDeviceToDevice, st));
    U.rows = (int)urows;
    U.cols = (int)d->n;
    U.nnz = d->q_nnz;
    U.ptr = su.ptr;
    U.idx = su.idx;
    U.val = su.val;
    Bump rest;
    rest.base = static_cast<char *>(scratch) + ((ub.used + 255) & ~size_t(255));
    rest.cap = scratch_bytes - ((ub.used + 255) & ~size_t(255));
    tm("Q_convert");
    rc = symmetrize_csr(ctx, U, p->sQ, p->Q, false, rest, &p->q_full_nnz, urow0, p->n0, p->n1);
    if (rc) return cleanup(rc);
    tm("Q_symmetrize_plan");
    if (sh && p->q_full_nnz != sh->q_local_nnz) return cleanup(fail(AQP_EINVAL, "q_local_nnz does not match the P block"));
    rc = split_q_diag(ctx, p, rest);
    if (rc) return cleanup(rc);
    tm("Q_split_diag_plan");
    if (n) AQP_CUDA(cudaMemcpyAsync(p->qd, d->q_diag, n * 8, cudaMemcpyDeviceToDevice, st));
    if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK && d->r_dense) {
      // full rows: the CSR values are R row-major (a shard: its columns
      // [n0,n1) of every row); check the implied pattern
      for (int64_t i = 0; i <= d->r_rows; ++i)
        if (host_r_indptr[i] != i * n) return cleanup(fail(AQP_EINVAL, "r_dense set but R rows are not full"));
      if (d->r_nnz != d->r_rows * n) return cleanup(fail(AQP_EINVAL, "r_dense: r_nnz != r_rows * n"));
      if (d->r_nnz) AQP_CUDA(cudaMemcpyAsync(p->sR.val, d->r_data, d->r_nnz * 8, cudaMemcpyDeviceToDevice, st));
      p->R.rows = (int)d->r_rows;
      p->R.cols = (int)n;
      p->R.nnz = d->r_nnz;
      p->R.val = p->sR.val;
      p->r_dense = 1;
    } else if (d->quad_kind == AQP_QUAD_SPARSE_LOW_RANK) {
      rc = upload_csr(ctx, p->sR, p->R, d->r_rows, d->n, d->r_indptr, d->r_indices, d->r_data, d->r_nnz,
                      host_r_indptr, false, p->bad);
      if (!rc) rc = transpose_csr(ctx, p->R, p->sRt, p->Rt, false, sc, p->n0, p->n1, 0, d->r_rows);
      if (!rc && p->Rt.nnz != d->r_nnz) rc = fail(AQP_EINVAL, "R block has columns outside [n0,n1)");
      if (rc) return cleanup(rc);
    }
  }
  if (n) {
    AQP_CUDA(cudaMemcpyAsync(p->c, d->cost, n * 8, cudaMemcpyDeviceToDevice, st));
    AQP_CUDA(cudaMemcpyAsync(p->vlo, d->var_lo, n * 8, cudaMemcpyDeviceToDevice, st));
    AQP_CUDA(cudaMemcpyAsync(p->vhi, d->var_hi, n * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (m) {
    AQP_CUDA(cudaMemcpyAsync(p->clo, d->con_lo, m * 8, cudaMemcpyDeviceToDevice, st));
    AQP_CUDA(cudaMemcpyAsync(p->chi, d->con_hi, m * 8, cudaMemcpyDeviceToDevice, st));
  }
  rc = build_cones(ctx, p->vlo, p->vhi, n, p->cone_r, p->recc_x, 0);
  if (!rc) rc = build_cones(ctx, p->clo, p->chi, m, p->cone_y, p->recc_s, 1);
  if (rc) return cleanup(rc);
  {  // SELL-32 layouts of the uniform matrices (filled by aqp_problem_attach_sell)
    CsrStore *stores[5] = {&p->sA, &p->sAt, &p->sQ, &p->sR, &p->sRt};
    DevCsr *mats[5] = {&p->A, &p->At, &p->Q, &p->R, &p->Rt};
    for (int i = 0; i < 5; ++i) {
      if (i == 2 && d->quad_kind == AQP_QUAD_DIAGONAL) continue;
      if (i >= 3 && (d->quad_kind != AQP_QUAD_SPARSE_LOW_RANK || p->r_dense)) continue;
      // pair layout for the non-symmetric matrices (A, A', R, R'), plain for Q
      rc = plan_sell(ctx, *mats[i], stores[i]->sell_off, stores[i]->sell_perm, i == 1, i != 2, sc,
                     &p->sell_total[i], &p->sell_sorted[i]);
      if (rc) return cleanup(rc);
    }
  }
  if (p->at_plan_deferred && !p->sell_sorted[1]) {  // no SELL-P for A': its CSR plan serves
    rc = plan_deferred_at(p);
    if (rc) return cleanup(rc);
  }
  int bad = 0;
  AQP_CUDA(cudaMemcpyAsync(&bad, p->bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  AQP_CUDA(cudaStreamSynchronize(st));
  tm("vectors_cones_sell_plan");
  if (bad) return cleanup(fail(AQP_EINVAL, "index out of range in CSR upload"));
  std::memset(&p->info, 0, sizeof(p->info));
  p->info.a_nnz = p->A.nnz;
  p->info.at_nnz = p->At.nnz;
  p->info.q_full_nnz = p->q_full_nnz;
  p->info.r_rows = d->r_rows;
  p->info.r_dense = p->r_dense;
  p->info.quad_kind = d->quad_kind;
  p->info.a_items = p->A.nitems;
  p->info.at_items = p->At.nitems;
  p->info.q_items = p->Q.nitems;
  p->info.persistent_bytes = b.used;
  *out = p;
  return AQP_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
// the banded ring path (AQP_RING=0 turns it off) for unsharded problems
static bool ring_on(const aqp_problem *p) {
  const char *e = getenv("AQP_RING");
  return p->nranks == 1 && !(e && e[0] == '0');
}

int aqp_problem_sell_bytes(const aqp_problem *p, size_t *bytes) {
  if (!p || !bytes) return fail(AQP_EINVAL, "NULL argument");
  size_t b = 0;
  for (int i = 0; i < 5; ++i)
    if (p->sell_total[i]) {
      b += align256((size_t)p->sell_total[i] * 4) + align256((size_t)p->sell_total[i] * 8);
      if (p->sell_sorted[i]) b += align256((size_t)(i == 0 ? p->A : i == 1 ? p->At : i == 2 ? p->Q : i == 3 ? p->R : p->Rt).rows);
    }
  if (ring_on(p))  // ring windows of A, A' and Q (which ops use them: AQP_RING_OFF)
    for (int i = 0; i < 3; ++i)
      if (p->sell_total[i]) b += align256((size_t)win_groups(i == 0 ? p->A : i == 1 ? p->At : p->Q) * sizeof(int2));
  *bytes = b;
  return AQP_OK;
}

int aqp_problem_attach_sell(aqp_problem *p, void *buf, size_t bytes) {
  if (!p) return fail(AQP_EINVAL, "NULL argument");
  size_t need = 0;
  AQP_TRY(aqp_problem_sell_bytes(p, &need));
  if (need == 0) return AQP_OK;
  if (!buf || bytes < need) return fail(AQP_ENOMEM, "SELL buffer too small (aqp_problem_sell_bytes)");
  AQP_CUDA(cudaSetDevice(p->ctx->device));
  cudaStream_t st = p->ctx->stream;
  CsrStore *stores[5] = {&p->sA, &p->sAt, &p->sQ, &p->sR, &p->sRt};
  DevCsr *mats[5] = {&p->A, &p->At, &p->Q, &p->R, &p->Rt};
  char *at = static_cast<char *>(buf);
  for (int i = 0; i < 5; ++i) {
    const int64_t tot = p->sell_total[i];
    if (!tot) continue;
    DevCsr &M = *mats[i];
    int *sidx = reinterpret_cast<int *>(at);
    at += align256((size_t)tot * 4);
    double *sval = reinterpret_cast<double *>(at);
    at += align256((size_t)tot * 8);
    if (p->sell_sorted[i]) {
      uint8_t *lens = reinterpret_cast<uint8_t *>(at);
      at += align256((size_t)M.rows);
      k_fill_sellp<<<(M.rows + 255) / 256, 256, 0, st>>>(M.ptr, M.idx, M.val, M.rows, stores[i]->sell_perm,
                                                         stores[i]->sell_off, sidx, sval, i != 2, lens);
      M.sell_len = lens;
      // the SELL-P kernel runs one block per 256 rows and sums long rows itself
      M.sell_perm = stores[i]->sell_perm;
      M.uniform = 1;
      M.nitems = (M.rows + kThreads - 1) / kThreads;
      M.smem_bytes = 0;
      if (i == 1) p->at_plan_deferred = false;  // the SELL-P plan replaces the CSR plan
    } else {
      k_fill_sell<<<(M.rows + 255) / 256, 256, 0, st>>>(M.ptr, M.idx, M.val, M.rows, stores[i]->sell_off, sidx,
                                                        sval, i != 2);
    }
    AQP_CUDA(cudaGetLastError());
    M.sell_off = stores[i]->sell_off;
    M.sell_idx = sidx;
    M.sell_val = sval;
  }
  p->info.ring_mask = 0;
  if (ring_on(p)) {
    for (int i = 0; i < 3; ++i) {
      DevCsr &M = *mats[i];
      if (!p->sell_total[i]) continue;
      int2 *win = reinterpret_cast<int2 *>(at);
      at += align256((size_t)win_groups(M) * sizeof(int2));
      if (!M.sell_idx || !(M.uniform || M.sell_perm) || M.row_off) continue;
      bool ok = false;
      AQP_TRY(plan_ring(p->ctx, M, win, ok));
      if (ok) {
        p->info.ring_mask |= 1 << i;
        M.win = win;
        M.win_groups = win_groups(M);
        M.win_rt = ring_rt();
        M.win_grid = std::min(p->ctx->sm_count * (kRingRT / M.win_rt), M.win_groups);
      }
    }
  }
  AQP_CUDA(cudaStreamSynchronize(st));
  p->info.a_items = p->A.nitems;
  p->info.at_items = p->At.nitems;
  p->info.q_items = p->Q.nitems;
  return AQP_OK;
}

int aqp_problem_get_info(const aqp_problem *p, aqp_problem_info *out) {
  if (!p || !out) return fail(AQP_EINVAL, "NULL argument");
  *out = p->info;
  return AQP_OK;
}

int aqp_problem_destroy(aqp_problem *p) {
  if (p)
    for (DevCsr *M : {&p->A, &p->At, &p->Q, &p->R, &p->Rt}) free_sell(*M, p->ctx->stream);
  delete p;
  return AQP_OK;
}

}  // extern "C"
