// aqp_common.cuh -- shared device/host helpers of libaqp.
//
// Arithmetic conventions (parity with the reference, anchorqp/_kernels/_core.pyx):
//  * the whole library is compiled with --fmad=false: every a*b+c is a rounded
//    multiply followed by a rounded add, exactly like the Cython kernels built
//    by gcc -O2 for baseline x86-64 (no FMA contraction);
//  * all reductions are deterministic: fixed per-thread order, fixed
//    shuffle tree, fixed cross-warp / cross-block order (no float atomics), so
//    a rerun reproduces every bit (reference tests/test_engine.py:307-314).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/aqp.h"

namespace aqp {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define AQP_CUDA(call)                                                             \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return ::aqp::fail(AQP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                        " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define AQP_TRY(call)             \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != AQP_OK) return rc_; \
  } while (0)

// ---------------------------------------------------------------- constants
constexpr int kThreads = 256;          // every kernel of the library uses 256-thread blocks
constexpr int kWarps = kThreads / 32;
constexpr int kTileNnz = 2048;         // nonzeros staged per SpMV row-block (16 KB + 8 KB smem)
constexpr int kSegNnz = 8192;          // nonzeros per block for a split long row
constexpr int kThreadRowMax = 48;      // longest row handled one-thread-per-row
constexpr int kMaxRed = 16;            // max reduction slots of one kernel
// ring path (spmv_ring_op): rows per group = threads per CTA, and the ring of
// cached columns of the gathered vector -- 1024 rows / 16384 columns (128 KB,
// one CTA per SM) or 512 rows / 12288 columns (96 KB, two CTAs per SM)
constexpr int kRingRT = 1024, kRingS = 16384;
constexpr int kRingRT2 = 512, kRingS2 = 12288;
__host__ __device__ constexpr int ring_cols(int rt) { return rt == kRingRT2 ? kRingS2 : kRingS; }

// ---------------------------------------------------------------- scalar helpers
// Reference semantics: _clip in _core.pyx:21-26 (lo first, then hi; NaN passes through)
__host__ __device__ __forceinline__ double clip(double v, double lo, double hi) {
  if (v < lo) return lo;
  if (v > hi) return hi;
  return v;
}

// Python's built-in max(a, b) / min(a, b): keep a unless b compares greater / smaller
__host__ __device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__host__ __device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// |x| by clearing the sign bit.  nvcc 12.9 -O3 miscompiles
// nanmax(0.0, fabs(d)) into `d > 0 ? |d| : 0` (SASS: DSETP.GTU on the
// un-abs'd operand), silently dropping negative residual components from
// every inf-norm (it also sees through a sign-bit mask).  An empty asm
// barrier makes the magnitude opaque, so no compare-with-zero rewrite can
// reach back to the signed operand.
__device__ __forceinline__ double absd(double x) {
  double r = fabs(x);
  asm volatile("" : "+d"(r));
  return r;
}

// numpy.max over nonnegative values with NaN propagation (np.abs(v).max())
__device__ __forceinline__ double nanmax(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return b > a ? b : a;
}

// cone projection, _core.pyx:95-115 (ZERO, NONNEG, NONPOS, FREE)
__device__ __forceinline__ double cone_proj(double v, int8_t code) {
  if (code == AQP_ZERO) return 0.0;
  if (code == AQP_NONNEG) return v > 0.0 ? v : 0.0;
  if (code == AQP_NONPOS) return v < 0.0 ? v : 0.0;
  return v;
}

// support_p term split (model.py:57-71): positive part against upper bound,
// negative part against lower bound; flag when a nonzero part meets an
// infinite bound of matching sign.
struct SupportAcc {
  double pos, neg, bad;
};
__device__ __forceinline__ void support_add(double z, double lo, double hi, double &pos, double &neg,
                                            double &bad) {
  if (z > 0.0) {
    if (isinf(hi)) bad = 1.0; else pos += hi * z;
  } else if (z < 0.0) {
    if (isinf(lo)) bad = 1.0; else neg += lo * z;
  }
}

// ---------------------------------------------------------------- deterministic reductions
template <int NS, int NM>
struct RedVals {
  double s[NS > 0 ? NS : 1];
  double m[NM > 0 ? NM : 1];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < NS; ++i) s[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NM; ++i) m[i] = 0.0;
  }
};

// Block reduction of NS sums and NM NaN-propagating maxes; result valid in
// thread 0.  Fixed xor-shuffle tree inside warps, then warp 0 folds the
// per-warp values in warp order.
template <int NS, int NM>
__device__ __forceinline__ void block_reduce(RedVals<NS, NM> &v, double *smem /* (blockDim/32)*(NS+NM) */) {
  constexpr int NT = NS + NM;
  if constexpr (NT == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int i = 0; i < NS; ++i) v.s[i] += __shfl_xor_sync(0xffffffffu, v.s[i], off);
#pragma unroll
    for (int i = 0; i < NM; ++i) v.m[i] = nanmax(v.m[i], __shfl_xor_sync(0xffffffffu, v.m[i], off));
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) smem[warp * NT + i] = v.s[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) smem[warp * NT + NS + i] = v.m[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // warps outer, slots inner: every slot still adds its warp values in
    // warp order (bitwise the slot-by-slot loop), but the NS + NM dependent
    // chains interleave instead of running back to back -- with 32 warps and
    // 7 slots that is 32 instead of 224 dependent shared-load + add steps
    // (the BB fold kernel's critical path, ~3.5 us, device trace)
    const int nw = (int)(blockDim.x >> 5);
#pragma unroll
    for (int i = 0; i < NS; ++i) v.s[i] = smem[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) v.m[i] = smem[NS + i];
    for (int w = 1; w < nw; ++w) {
#pragma unroll
      for (int i = 0; i < NS; ++i) v.s[i] += smem[w * NT + i];
#pragma unroll
      for (int i = 0; i < NM; ++i) v.m[i] = nanmax(v.m[i], smem[w * NT + NS + i]);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- row shards over peer memory
// Multi-GPU: rank r stores and owns rows [n0,n1) of A' and
// Q (x side) and rows [m0,m1) of A (y side).  Every vector that an SpMV
// gathers lives in a per-rank WINDOW [xw0, xw1) / [yw0, yw1) covering the
// rank's own rows and every column its rows gather (column indices stay
// global: a kernel gathers through base - xw0).  The kernel that produces a
// rank's slice stores it locally AND into every peer's window that contains
// the entry (NVLink P2P stores into the peers' solver workspaces; the
// exchange regions have the identical layout on every rank -- buffers are
// sized by max-over-ranks capacities -- so the peer address of entry g is
// local address + delta[k] + 8 (xw0_self - xw0_k), precomputed per side as
// xdelta / ydelta).  Reductions and barriers are one-block mailbox
// exchanges: each rank writes its block-folded partials into
// mail[epoch & 1][rank] of every peer, then releases flag[rank] = epoch on
// every peer and acquires all flags >= epoch; every rank then combines the P
// partials in rank order, so all ranks hold bitwise-identical scalars and
// take identical branches (the CUDA-graph conditionals included).  No NCCL
// call sits on the data path.
constexpr int kMaxRanks = 8;
constexpr int kMaxVec = 256;  // longest vector all-reduce (R x of a row-sharded low-rank Q)

struct CommBlock {
  unsigned long long flag[kMaxRanks];  // flag[k]: last epoch rank k arrived at (written by rank k)
  unsigned long long epoch;            // this rank's exchange counter (device-owned)
  unsigned long long err;              // epoch of an exchange whose wait timed out (0 = none)
  unsigned long long pad[6];
  double mail[2][kMaxRanks][kMaxRed];
  double vmail[2][kMaxRanks][kMaxVec];  // vector all-reduce (comm_allreduce_vec)
};

struct Comm {
  int rank = 0, nranks = 1;
  CommBlock *cb = nullptr;
  unsigned long long timeout_ns = 30000000000ull;  // a peer that never arrives: give up, flag, carry on
  long long delta[kMaxRanks] = {};  // byte offset local -> rank k's mapping of the same buffer
  // ... of an x-side / y-side gathered entry (the windows start at different
  // global indices on different ranks): delta[k] + 8 (w0_self - w0_k)
  long long xdelta[kMaxRanks] = {}, ydelta[kMaxRanks] = {};
  // Halo ranges: rank k only ever gathers x entries in [xlo[k], xhi[k]) (the
  // columns of its rows of A and Q) and y entries in [ylo[k], yhi[k]) (the
  // columns of its rows of A'), so a producer stores to peer k only what
  // falls in k's range -- for a banded C5 that is a boundary strip instead of
  // the whole slice.  Defaults: the windows.
  long long xlo[kMaxRanks] = {}, xhi[kMaxRanks] = {}, ylo[kMaxRanks] = {}, yhi[kMaxRanks] = {};
};

// c.delta[k] for a run-time k without indexing the kernel-parameter array
// dynamically (that would copy the whole op into local memory)
__device__ __forceinline__ long long peer_delta(const Comm &c, int k) {
  long long d = 0;
#pragma unroll
  for (int j = 0; j < kMaxRanks; ++j)
    if (j == k) d = c.delta[j];
  return d;
}
template <class T>
__device__ __forceinline__ T *peer_addr(const Comm &c, T *p, int k) {
  return reinterpret_cast<T *>(reinterpret_cast<char *>(p) + peer_delta(c, k));
}

// store `val` (local entry p[i], global index g) into the window of every
// peer that gathers g (x side: side = 0, y side: 1); the local store is the
// caller's
__device__ __forceinline__ void peer_put_halo(const Comm &c, int side, double *p, int64_t i, int64_t g, double val) {
  if (c.nranks <= 1) return;
#pragma unroll
  for (int k = 0; k < kMaxRanks; ++k) {
    const long long lo = side ? c.ylo[k] : c.xlo[k], hi = side ? c.yhi[k] : c.xhi[k];
    if (k < c.nranks && k != c.rank && g >= lo && g < hi)
      *reinterpret_cast<double *>(reinterpret_cast<char *>(p + i) + (side ? c.ydelta[k] : c.xdelta[k])) = val;
  }
}

__device__ __forceinline__ unsigned long long global_ns_() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide (every thread of the block calls it): all-reduce of thread 0's
// `a` over the ranks, combined in rank order; result in thread 0.  With NS =
// NM = 0 it is a pure barrier.  No-op for one rank.
template <int NS, int NM>
__device__ __forceinline__ void comm_allreduce(RedVals<NS, NM> &a, const Comm &c) {
  if (c.nranks <= 1) return;
  constexpr int NT = NS + NM;
  constexpr int NTA = NT > 0 ? NT : 1;
  __shared__ unsigned long long s_epoch;
  __shared__ double s_mine[NTA];
  __shared__ double s_all[kMaxRanks * NTA];
  if (threadIdx.x == 0) {
    const unsigned long long e = c.cb->epoch + 1;
    c.cb->epoch = e;
    s_epoch = e;
#pragma unroll
    for (int i = 0; i < NS; ++i) s_mine[i] = a.s[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) s_mine[NS + i] = a.m[i];
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int P = c.nranks;
  if (NT > 0) {
    for (int t = threadIdx.x; t < P * NT; t += blockDim.x) {
      const int k = t / NTA, i = t % NTA;
      *peer_addr(c, &c.cb->mail[e & 1][c.rank][i], k) = s_mine[i];
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < P) {
    __threadfence_system();
    st_release_sys(peer_addr(c, &c.cb->flag[c.rank], (int)threadIdx.x), e);
    // bounded wait: a lost peer must not hang the GPU; the host turns the
    // recorded epoch into a DeviceError at its next sync (aqp_solver_*)
    const unsigned long long t0 = global_ns_();
    const bool broken = *(volatile unsigned long long *)&c.cb->err != 0;  // fail fast after a loss
    while (!broken && ld_acquire_sys(&c.cb->flag[threadIdx.x]) < e) {
      __nanosleep(64);
      if (global_ns_() - t0 > c.timeout_ns) {
        atomicCAS(&c.cb->err, 0ull, e);
        break;
      }
    }
  }
  __syncthreads();
  if (NT > 0) {
    for (int t = threadIdx.x; t < P * NT; t += blockDim.x) {
      const int k = t / NTA, i = t % NTA;
      s_all[t] = __ldcv(&c.cb->mail[e & 1][k][i]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        double v = s_all[i];
        for (int k = 1; k < P; ++k) v += s_all[k * NTA + i];
        a.s[i] = v;
      }
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        double v = s_all[NS + i];
        for (int k = 1; k < P; ++k) v = nanmax(v, s_all[k * NTA + NS + i]);
        a.m[i] = v;
      }
    }
    __syncthreads();
  }
}

// Block-wide: in-place all-reduce (sum over ranks, combined in rank order)
// of the `len` (<= kMaxVec) doubles at v; every thread of the block calls it.
// All ranks end with bitwise-identical sums.  No-op for one rank.
__device__ __forceinline__ void comm_allreduce_vec(double *v, int len, const Comm &c) {
  if (c.nranks <= 1) return;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    const unsigned long long e = c.cb->epoch + 1;
    c.cb->epoch = e;
    s_epoch = e;
  }
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int P = c.nranks;
  for (int t = threadIdx.x; t < P * len; t += blockDim.x) {
    const int k = t / len, i = t % len;
    *peer_addr(c, &c.cb->vmail[e & 1][c.rank][i], k) = v[i];
  }
  __syncthreads();
  if ((int)threadIdx.x < P) {
    __threadfence_system();
    st_release_sys(peer_addr(c, &c.cb->flag[c.rank], (int)threadIdx.x), e);
    const unsigned long long t0 = global_ns_();
    const bool broken = *(volatile unsigned long long *)&c.cb->err != 0;
    while (!broken && ld_acquire_sys(&c.cb->flag[threadIdx.x]) < e) {
      __nanosleep(64);
      if (global_ns_() - t0 > c.timeout_ns) {
        atomicCAS(&c.cb->err, 0ull, e);
        break;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    double a = __ldcv(&c.cb->vmail[e & 1][0][i]);
    for (int k = 1; k < P; ++k) a += __ldcv(&c.cb->vmail[e & 1][k][i]);
    v[i] = a;
  }
  __syncthreads();
}

// Grid-level epilogue: see grid_end / fin_op in aqp_kernels.cuh.
struct GridRed {
  double *partials;     // >= kMaxRed * gridDim.x doubles, layout [slot][block]
  unsigned int *ticket;  // zero between launches (reset by the last block)
  Comm comm;            // row shards: grid totals are all-reduced over the ranks
  // optional device trace (AQP_TRACE=1): (tag, globaltimer ns) pairs
  unsigned long long *trace = nullptr;
  unsigned int *trace_n = nullptr;
  unsigned int trace_cap = 0;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// tag = kind << 32 | grid size (kind 0 spmv, 1 elem, 2 fin start, 3 fin end)
__device__ __forceinline__ void trace_mark(const GridRed &g, unsigned kind) {
  if (g.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned i = atomicAdd(g.trace_n, 1u) % g.trace_cap;
    g.trace[2 * i] = ((unsigned long long)kind << 32) | gridDim.x;
    g.trace[2 * i + 1] = global_ns();
  }
}

// ---------------------------------------------------------------- SpMV work partition
// One block per item.  THREAD: rows [row0,row1) whose nonzeros [k0,k1) fit
// one smem tile, one thread per row, row sum sequential in column order
// (bitwise the Cython order).  WARP: same tile, one warp per row (used when
// rows are long enough that a sequential chain would be latency bound).
// LONG: segment `seg` of `nseg` of one row longer than a tile.  LONGSEQ
// (strict plans only): a long row summed by one thread in column order.
// STAGED: a THREAD item whose nonzeros ([k0,k1) <= one tile) are first staged
// as products in shared memory with coalesced index/value loads and one
// parallel burst of gathers, then summed one thread per row in column order
// (bitwise the THREAD order); chosen for matrices whose rows are long enough
// that the THREAD item's strided per-row loads cost more L1 wavefronts than
// the staging barrier (mean row length >= AQP_STAGED_MIN, default 8).
enum : int { kItemThread = 0, kItemWarp = 1, kItemLong = 2, kItemLongSeq = 3, kItemStaged = 4 };

struct __align__(16) PlanItem {
  int row0, row1, k0, k1;
  int kind, seg, nseg, segbase;
};

// SELL-32 element position of nonzero k of the row at SELL position p:
// `off` = the slice's offset (sell_off[p / 32]), lane = p % 32.  Pair layout
// (the non-symmetric A / A' / R / R'): [k0 k1 of lane 0, k0 k1 of lane 1, ...] per
// pair of steps, even slice widths -- one 128-bit load fetches a lane's two
// values and one 64-bit load its two column indices (C5-shaped A' / A passes
// 4-5% faster).  Plain layout (Q): k-major, one entry per lane -- the pair
// layout made the 4-nonzero rows of the gradient pass 20% slower.
__host__ __device__ __forceinline__ int64_t sell_pos(int64_t off, int lane, int k, bool pair) {
  return pair ? off + 64 * (int64_t)(k >> 1) + 2 * lane + (k & 1) : off + 32 * (int64_t)k + lane;
}
__host__ __device__ __forceinline__ int64_t sell_width(int longest, bool pair) {  // entries per slice
  return 32 * (int64_t)(pair ? (longest + 1) & ~1 : longest);
}

// device CSR with int32 indices plus its work plan
struct DevCsr {
  int rows = 0, cols = 0;
  int64_t nnz = 0;
  const int *ptr = nullptr;
  const int *idx = nullptr;
  const double *val = nullptr;
  const PlanItem *plan = nullptr;
  int nitems = 0;
  int nlongseg = 0;
  double *seg_part = nullptr;          // 2 * nlongseg doubles
  unsigned int *seg_ticket = nullptr;  // nlongseg counters
  int smem_bytes = 0;                  // dynamic shared memory per block (WARP items only)
  int uniform = 0;                     // every item is THREAD over rows [256 b, 256 b + 256)
  int row_off = 0;                     // global index of local row 0 (row shards of a symmetric Q)
  // SELL-32 copy of a uniform (THREAD-only) plan's matrix: the k-th nonzero of
  // row r sits at sell_off[r / 32] + 32 k + r % 32, so the warp's k-th loads
  // (one row per lane) are coalesced -- one L1 wavefront for 32 indices
  // instead of ~5 for the strided CSR rows.  Same nonzeros, same order per row.
  // (non-symmetric matrices: pair layout -- a lane's nonzeros 2j, 2j+1 are
  // adjacent, so one 128-bit load fetches two values and one 64-bit load two
  // column indices; the warp still reads contiguous 512 B / 256 B per pair
  // step; see sell_pos)
  const int64_t *sell_off = nullptr;
  const int *sell_idx = nullptr;
  const double *sell_val = nullptr;
  // SELL-P (block-sorted SELL, for the A' of banded problems): within every
  // 256-row block the rows are ordered by length (descending, stable), and
  // the SELL-32 slices run over those sorted POSITIONS -- position p holds
  // row (p & ~255) + sell_perm[p] -- so a slice's rows have near-equal
  // lengths (1.12x padding on C5's A' instead of 1.72x).  Rows longer than
  // kThreadRowMax are not in the slices (the block sums them together).  Row
  // sums stay sequential per row; the epilogue runs in natural row order after
  // a shared-memory hand-off.  (Sorting within a warp only -- no block
  // barrier, natural slice widths -- measured slower: C5 A' 2.80 ms.)
  const uint8_t *sell_perm = nullptr;
  // SELL-P: the length of the row at each sorted position (255: longer), so a
  // thread starts its slice loads after one round trip instead of three
  // (position -> row -> row pointers)
  const uint8_t *sell_len = nullptr;
  // full symmetric Q of a uniform plan: its diagonal moved out of the CSR into
  // diag[local row].  A row's upper sum starts with diag * x[row] -- the
  // diagonal is the first j >= i entry, so the order is unchanged -- and the
  // CSR loop is one nonzero (often one gather batch) shorter.
  const double *diag = nullptr;
  // banded ring path (spmv_ring_op, unsharded SELL / SELL-P matrices whose
  // nonzeros stay within a moving column window): per group of kRingRT rows
  // the column window [x, y] its rows gather, made monotone (x: suffix
  // minimum, y: prefix maximum); null when the band does not fit the ring
  const int2 *win = nullptr;
  int win_groups = 0;
  int win_rt = 0;    // rows per group (kRingRT or kRingRT2)
  int win_grid = 0;  // persistent grid: the CTAs resident at once
};

}  // namespace aqp
