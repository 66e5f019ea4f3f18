// aqp_kernels.cuh -- the kernel skeletons every op of libaqp is built from.
//
//   spmv_op<Op>: one pass over a CSR matrix (A, A', the full symmetric Q or
//     P) with the op's per-row epilogue fused in and up to kMaxRed
//     deterministic reductions.
//   elem_op<Op>: one fixed-grid pass over a vector index space, same tail.
//   fin_op<Op>:  a single block that folds the partials of the preceding
//     spmv_op/elem_op launch and runs the op's scalar `finalize` (e.g. the
//     BB step-size rule and the CUDA-graph loop condition).
//
// Reductions end in one of two ways.  Hot ops (Op::SPLIT = true: the BB
// gradient pass, the primal/dual epilogues) only publish per-block partials
// and leave the fold to a fin_op node that follows in the graph -- measured on
// C2, a last-block ticket (fence + atomic before every block retires) costs
// ~14 us per launch, a one-block fin kernel ~3 us.  Cold ops (the
// certification kernels) keep the last-block ticket.
//
// Row work of an SpMV is cut into plan items (aqp_problem.cu):
//   THREAD  <= 256 short rows, one thread per row, the row's nonzeros read
//           straight from HBM in column order (bitwise the Cython order);
//           the row's epilogue operands are loaded first (Op::RowIn) so their
//           latency overlaps the index -> gather chain;
//   WARP    rows of medium length staged in shared memory, one warp per row;
//   LONG    one segment of a row longer than a tile (block reduction, the
//           last segment block combines the row);
//   LONGSEQ (strict plans) a long row summed sequentially by one thread.
//
// Op concept:
//   static constexpr int NS, NM;       number of sums / NaN-propagating maxes
//   static constexpr bool SYM;         (spmv) full symmetric matrix: the row sum
//                                      is (sum of j<r entries) + (sum of j>=r),
//                                      each sequential -- bitwise the order of
//                                      _core.pyx:62-80 sym_matvec
//   static constexpr bool FINAL;       run finalize() after the grid is done
//   [static constexpr bool SPLIT;]     finalize in a separate fin_op launch
//   bool skip() const;                 uniform early exit (e.g. halted window)
//   void prepare();                    per-thread setup on a private copy of the
//                                      op (resolves device-side slot indices)
//   double gather(int col) const;      (spmv) source vector entry
//   void row(int r, double v, RedVals&) const;   (spmv) epilogue for row r
//   [struct RowIn; RowIn load_row(int r) const;
//    void row_in(int r, double v, const RowIn&, RedVals&) const;]
//   void elem(int64_t i, RedVals&) const;        (elem)
//   void finalize(const RedVals&) const;         one thread, after the fold
#pragma once

#include <type_traits>

#include "aqp_common.cuh"

#ifndef AQP_UNIFORM_MIN_BLOCKS
#define AQP_UNIFORM_MIN_BLOCKS 4
#endif
#ifndef AQP_SPMV_MIN_BLOCKS
#define AQP_SPMV_MIN_BLOCKS 4
#endif

namespace aqp {

// Programmatic dependent launch (PDL).  Graph edges between consecutive
// kernel nodes are programmatic: a kernel may be scheduled while its
// predecessor drains; it reads nothing the predecessor produces before
// pdl_wait() (griddepcontrol.wait: full completion + memory flush of the
// predecessor), and releases its own dependents with pdl_trigger() once its
// main work is issued.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct NoRowIn {};
template <class Op, class = void>
struct RowInOf {
  using type = NoRowIn;
  static constexpr bool value = false;
};
template <class Op>
struct RowInOf<Op, std::void_t<typename Op::RowIn>> {
  using type = typename Op::RowIn;
  static constexpr bool value = true;
};

// Per-op tuning of the uniform (THREAD-only) SpMV instantiation:
//   Op::ROWIN_LATE    load the row's epilogue operands after the gathers
//                     (frees registers during the gather chain)
//   Op::UNIFORM_BLOCKS resident 256-thread blocks per SM the register budget
//                     targets (occupancy vs. per-thread batching)
// Measured on C2 (scripts/kern_variants.sh): the BB gradient pass is fastest
// late/6 (50 us vs 56 us early/4), the dual pass P2 early/4.
template <class Op, class = void>
struct RowInLateOf {
  static constexpr bool value = false;
};
template <class Op>
struct RowInLateOf<Op, std::void_t<decltype(Op::ROWIN_LATE)>> {
  static constexpr bool value = Op::ROWIN_LATE;
};
template <class Op, class = void>
struct UniformBlocksOf {
  static constexpr int value = AQP_UNIFORM_MIN_BLOCKS;
};
template <class Op>
struct UniformBlocksOf<Op, std::void_t<decltype(Op::UNIFORM_BLOCKS)>> {
  static constexpr int value = Op::UNIFORM_BLOCKS;
};

template <class Op, class = void>
struct SplitOf {
  static constexpr bool value = false;
};
template <class Op>
struct SplitOf<Op, std::void_t<decltype(Op::SPLIT)>> {
  static constexpr bool value = Op::SPLIT;
};

// Fold per-block partials stored [slot][block] in block order (thread t takes
// blocks t, t+256, ... with loads batched four blocks at a time), then the
// fixed tree.  Result in thread 0.
template <int NS, int NM>
__device__ __forceinline__ void fold_partials(RedVals<NS, NM> &a, const double *partials, unsigned nb,
                                              double *smem) {
  constexpr int NT = NS + NM;
  a.zero();
  if constexpr (NT > 0) {
    constexpr int U = 4;
    const unsigned nt = blockDim.x;
    for (unsigned b0 = threadIdx.x; b0 < nb; b0 += U * nt) {
      double t[U][NT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned b = b0 + u * nt;
#pragma unroll
        for (int i = 0; i < NT; ++i) t[u][i] = b < nb ? partials[(size_t)i * nb + b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int i = 0; i < NS; ++i) a.s[i] += t[u][i];
#pragma unroll
        for (int i = 0; i < NM; ++i) a.m[i] = nanmax(a.m[i], t[u][NS + i]);
      }
    }
  }
  block_reduce<NS, NM>(a, smem);
}

// End of a reducing launch.  SPLIT: publish this block's partials and return
// false.  Otherwise the last-block ticket: returns true in thread 0 of the
// last block with the grid totals in `v`.
template <int NS, int NM, bool SPLIT>
__device__ __forceinline__ bool grid_end(RedVals<NS, NM> &v, GridRed g, double *smem) {
  constexpr int NT = NS + NM;
  __shared__ bool last;
  const unsigned slot = blockIdx.x;
  if constexpr (NT > 0) block_reduce<NS, NM>(v, smem);
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
#pragma unroll
    for (int i = 0; i < NS; ++i) g.partials[(size_t)i * nb + slot] = v.s[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) g.partials[(size_t)(NS + i) * nb + slot] = v.m[i];
    if (!SPLIT) {
      // only thread 0 published, so only thread 0 fences
      __threadfence();
      last = (atomicAdd(g.ticket, 1u) == nb - 1);
      if (last) __threadfence();
    }
  }
  if (SPLIT) return false;
  __syncthreads();
  if (!last) return false;
  RedVals<NS, NM> a;
  fold_partials<NS, NM>(a, g.partials, gridDim.x, smem);
  comm_allreduce<NS, NM>(a, g.comm);
  v = a;
  if (threadIdx.x == 0) *g.ticket = 0u;
  return threadIdx.x == 0;
}

#ifndef AQP_SPMV_MIN_BLOCKS
#define AQP_SPMV_MIN_BLOCKS 4
#endif
#ifndef AQP_GATHER_BATCH
#define AQP_GATHER_BATCH 4
#endif
#ifndef AQP_SELL_BATCH  // nonzeros per load batch on the SELL paths
#define AQP_SELL_BATCH AQP_GATHER_BATCH
#endif

// Load the SELL entries k .. k+AQP_SELL_BATCH-1 of one row (lane `lane` of
// the slice at `off`) into cc / pv; entries past `len` are not used.  PAIR:
// the pair layout (non-symmetric matrices) -- two 128-bit value loads and two
// 64-bit index loads per batch of 4.  The layout follows the matrix kind and
// so the op: every non-symmetric matrix (A, A', R, R') is stored in pairs,
// the symmetric Q plainly, so PAIR = !Op::SYM is a compile-time choice (a
// runtime flag cost 2-7% on every pass: code and registers for both paths).
template <bool PAIR>
__device__ __forceinline__ void sell_load(const DevCsr &M, int64_t off, int lane, int k, int len,
                                          int (&cc)[AQP_SELL_BATCH], double (&pv)[AQP_SELL_BATCH]) {
  static_assert(AQP_SELL_BATCH % 2 == 0, "the pair layout loads whole pairs");
  if constexpr (PAIR) {
#pragma unroll
    for (int h = 0; h < AQP_SELL_BATCH / 2; ++h) {
      const int kk = k + 2 * h;
      if (kk < len) {
        const int64_t q = sell_pos(off, lane, kk, true);
        const int2 ci = __ldg(reinterpret_cast<const int2 *>(M.sell_idx + q));
        const double2 vv = __ldg(reinterpret_cast<const double2 *>(M.sell_val + q));
        cc[2 * h] = ci.x;
        cc[2 * h + 1] = ci.y;
        pv[2 * h] = vv.x;
        pv[2 * h + 1] = vv.y;
      } else {
        cc[2 * h] = cc[2 * h + 1] = 0;
        pv[2 * h] = pv[2 * h + 1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < AQP_SELL_BATCH; ++u) {
      const bool in = k + u < len;
      cc[u] = in ? __ldg(M.sell_idx + sell_pos(off, lane, k + u, false)) : 0;
      pv[u] = in ? __ldg(M.sell_val + sell_pos(off, lane, k + u, false)) : 0.0;
    }
  }
}

// UNIFORM: the plan is all THREAD items over [256 b, 256 b + 256) (the common
// case of short-row matrices, e.g. every C2 pass); the instantiation then
// carries only the thread-per-row path, which needs far fewer registers
// Stage the products of one tile [k0, k1) (<= kTileNnz nonzeros) into shared
// memory (sprod, and scol for a symmetric row split): thread t takes nonzeros
// t, t + 256, ..., so each warp-wide load and gather covers 32 consecutive
// nonzeros.  (128-bit int4 / double2 staging was measured 10% slower on the C5
// A' pass: a warp's gather then spans 4x the nonzeros, i.e. more cache lines.)
template <class Op>
__device__ __forceinline__ void stage_tile(const DevCsr &M, int k0, int k1, const Op &o, double *sprod, int *scol) {
  int cs[kTileNnz / kThreads];
#pragma unroll
  for (int u = 0; u < kTileNnz / kThreads; ++u) {
    const int k = k0 + threadIdx.x + u * kThreads;
    cs[u] = k < k1 ? __ldg(M.idx + k) : 0;
  }
#pragma unroll
  for (int u = 0; u < kTileNnz / kThreads; ++u) {
    const int k = k0 + threadIdx.x + u * kThreads;
    if (k < k1) {
      sprod[k - k0] = __ldg(M.val + k) * o.gather(cs[u]);
      if constexpr (Op::SYM) scol[k - k0] = cs[u];
    }
  }
}

// One plan item of an SpMV pass with op `o`: the block's rows are summed
// (THREAD / STAGED / WARP / LONGSEQ / LONG, see the file header) and their
// epilogue accumulates into `acc`.  Shared by spmv_op (one item per block) and
// the persistent small-problem window kernel (items looped over a resident grid).
template <class Op, bool UNIFORM>
__device__ __forceinline__ void spmv_item(const DevCsr &M, const PlanItem &it, const Op &o,
                                          RedVals<Op::NS, Op::NM> &acc, double *sprod, int *scol, double *sred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (it.kind == kItemThread) {
    // one thread per row, straight from HBM (no staging, no barrier)
    const int r = it.row0 + threadIdx.x;
    if (r < it.row1) {
      using RowIn = typename RowInOf<Op>::type;
      RowIn rin{};
      if constexpr (RowInOf<Op>::value && !RowInLateOf<Op>::value) rin = o.load_row(r);
      const int b = __ldg(M.ptr + r), e = __ldg(M.ptr + r + 1);
      const int rg = r + M.row_off;  // global row (diagonal position of a symmetric shard)
      double lo = 0.0, up = 0.0;
      if (Op::SYM && M.diag) up = __ldg(M.diag + r) * o.gather(rg);  // split diagonal, first of the j >= i sum
      if ((UNIFORM || M.uniform) && M.sell_idx) {
        // SELL-32: the warp's k-th nonzeros are contiguous (coalesced loads)
        const int len = e - b;
        if constexpr (!Op::SYM) {  // pair layout (A, A', R, R')
          const int64_t soff = __ldg(M.sell_off + (r >> 5));
          for (int k = 0; k < len; k += AQP_SELL_BATCH) {
            int cc[AQP_SELL_BATCH];
            double pv[AQP_SELL_BATCH];
            sell_load<true>(M, soff, r & 31, k, len, cc, pv);
#pragma unroll
            for (int u = 0; u < AQP_SELL_BATCH; ++u)
              if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
            for (int u = 0; u < AQP_SELL_BATCH; ++u)
              if (k + u < len) up += pv[u];
          }
        } else {  // plain layout (Q); written out here: this schedule is the
                  // gradient pass's best (the shared loader cost it 7%)
          const int64_t base = __ldg(M.sell_off + (r >> 5)) + (r & 31);
          for (int k = 0; k < len; k += AQP_SELL_BATCH) {
            int cc[AQP_SELL_BATCH];
            double pv[AQP_SELL_BATCH];
#pragma unroll
            for (int u = 0; u < AQP_SELL_BATCH; ++u) {
              const bool in = k + u < len;
              cc[u] = in ? __ldg(M.sell_idx + base + 32 * (k + u)) : 0;
              pv[u] = in ? __ldg(M.sell_val + base + 32 * (k + u)) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < AQP_SELL_BATCH; ++u)
              if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
            for (int u = 0; u < AQP_SELL_BATCH; ++u) {
              if (k + u < len) {
                if (Op::SYM && cc[u] < rg) lo += pv[u]; else up += pv[u];
              }
            }
          }
        }
      } else {
#if AQP_GATHER_BATCH > 1
      // the row's nonzeros in chunks of AQP_GATHER_BATCH: all index/value
      // loads of a chunk, then all its gathers, then the sums in column
      // order (bitwise the sequential loop) -- two dependent round trips per
      // chunk instead of two per nonzero
      for (int k = b; k < e; k += AQP_GATHER_BATCH) {
        int cc[AQP_GATHER_BATCH];
        double pv[AQP_GATHER_BATCH];
#pragma unroll
        for (int u = 0; u < AQP_GATHER_BATCH; ++u) {
          const bool in = k + u < e;
          cc[u] = in ? __ldg(M.idx + k + u) : 0;
          pv[u] = in ? __ldg(M.val + k + u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < AQP_GATHER_BATCH; ++u)
          if (k + u < e) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
        for (int u = 0; u < AQP_GATHER_BATCH; ++u) {
          if (k + u < e) {
            if (Op::SYM && cc[u] < rg) lo += pv[u]; else up += pv[u];
          }
        }
      }
#else
      for (int k = b; k < e; ++k) {
        const int c = __ldg(M.idx + k);
        const double p = __ldg(M.val + k) * o.gather(c);
        if (Op::SYM && c < rg) lo += p; else up += p;
      }
#endif
      }
      const double val = Op::SYM ? lo + up : up;
      if constexpr (RowInOf<Op>::value && RowInLateOf<Op>::value) rin = o.load_row(r);
      if constexpr (RowInOf<Op>::value) o.row_in(r, val, rin, acc); else o.row(r, val, acc);
    }
  } else if (UNIFORM) {
    // not reached: uniform plans hold THREAD items only
  } else if (it.kind == kItemWarp) {
    // rows of medium length: stage the tile's products with coalesced loads,
    // then one warp per row (tree order, deterministic)
    const int k0 = it.k0, k1 = it.k1;
    stage_tile(M, k0, k1, o, sprod, scol);
    __syncthreads();
    for (int r = it.row0 + warp; r < it.row1; r += kWarps) {
      const int b = __ldg(M.ptr + r) - k0, e = __ldg(M.ptr + r + 1) - k0;
      double lo = 0.0, up = 0.0;
      for (int j = b + lane; j < e; j += 32) {
        if (Op::SYM && scol[j] < r + M.row_off) lo += sprod[j]; else up += sprod[j];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        up += __shfl_xor_sync(0xffffffffu, up, off);
        if constexpr (Op::SYM) lo += __shfl_xor_sync(0xffffffffu, lo, off);
      }
      if (lane == 0) o.row(r, Op::SYM ? lo + up : up, acc);
    }
  } else if (it.kind == kItemStaged) {
    // products staged with coalesced loads and one burst of gathers, then
    // one thread per row sums its slice of the tile in column order
    const int k0 = it.k0, k1 = it.k1;
    const int r = it.row0 + threadIdx.x;
    const bool has = r < it.row1;
    using RowIn = typename RowInOf<Op>::type;
    RowIn rin{};
    int b = 0, e = 0;
    if (has) {
      if constexpr (RowInOf<Op>::value) rin = o.load_row(r);  // early: measured best for STAGED
      b = __ldg(M.ptr + r) - k0;
      e = __ldg(M.ptr + r + 1) - k0;
    }
    stage_tile(M, k0, k1, o, sprod, scol);
    __syncthreads();
    if (has) {
      const int rg = r + M.row_off;
      double lo = 0.0, up = 0.0;
      for (int j = b; j < e; ++j) {
        if (Op::SYM && scol[j] < rg) lo += sprod[j]; else up += sprod[j];
      }
      const double val = Op::SYM ? lo + up : up;
      if constexpr (RowInOf<Op>::value) o.row_in(r, val, rin, acc); else o.row(r, val, acc);
    }
  } else if (it.kind == kItemLongSeq) {
    if (threadIdx.x == 0) {
      const int r = it.row0;
      double lo = 0.0, up = 0.0;
      for (int k = it.k0; k < it.k1; ++k) {
        const int c = __ldg(M.idx + k);
        const double p = __ldg(M.val + k) * o.gather(c);
        if (Op::SYM && c < r + M.row_off) lo += p; else up += p;
      }
      o.row(r, Op::SYM ? lo + up : up, acc);
    }
  } else {
    // one segment of a long row: strided per-thread sums, fixed tree, then
    // (if split) the last segment block folds the segment partials in order
    const int r = it.row0;
    RedVals<2, 0> lu;
    lu.zero();
    for (int k = it.k0 + threadIdx.x; k < it.k1; k += kThreads) {
      const int c = __ldg(M.idx + k);
      const double p = __ldg(M.val + k) * o.gather(c);
      if (Op::SYM && c < r + M.row_off) lu.s[0] += p; else lu.s[1] += p;
    }
    block_reduce<2, 0>(lu, sred);
    if (it.nseg == 1) {
      if (threadIdx.x == 0) o.row(r, Op::SYM ? lu.s[0] + lu.s[1] : lu.s[1], acc);
    } else {
      __shared__ bool lastseg;
      if (threadIdx.x == 0) {
        M.seg_part[2 * (it.segbase + it.seg)] = lu.s[0];
        M.seg_part[2 * (it.segbase + it.seg) + 1] = lu.s[1];
        __threadfence();
        lastseg = (atomicAdd(M.seg_ticket + it.segbase, 1u) == (unsigned)(it.nseg - 1));
        if (lastseg) __threadfence();
      }
      __syncthreads();
      if (lastseg && threadIdx.x == 0) {
        double lo = 0.0, up = 0.0;
        for (int s = 0; s < it.nseg; ++s) {
          lo += __ldcg(M.seg_part + 2 * (it.segbase + s));
          up += __ldcg(M.seg_part + 2 * (it.segbase + s) + 1);
        }
        M.seg_ticket[it.segbase] = 0u;
        o.row(r, Op::SYM ? lo + up : up, acc);
      }
    }
  }
}

// One 256-row block of a SELL-P matrix (DevCsr::sell_perm): thread t sums
// the row at sorted position t from the SELL slices (coalesced index / value
// loads, the row's nonzeros in column order), the block sums its long rows
// together (tree order, like the WARP / LONG items), the sums meet in shared
// memory, and thread t runs the epilogue of row 256 b + t -- the same row ->
// thread map (so the same reductions) as the natural uniform path.
template <class Op>
__device__ __forceinline__ void spmv_sellp_block(const DevCsr &M, const Op &o, RedVals<Op::NS, Op::NM> &acc,
                                                 double *sred) {
  __shared__ double ssum[kThreads];
  __shared__ int lrow[kThreads];
  __shared__ int nlr;
  const int blk = blockIdx.x * kThreads, t = threadIdx.x;
  const int rn = blk + t;  // epilogue row (= sorted position index)
  using RowIn = typename RowInOf<Op>::type;
  RowIn rin{};
  const bool has = rn < M.rows;
  if constexpr (RowInOf<Op>::value && !RowInLateOf<Op>::value)
    if (has) rin = o.load_row(rn);
  const int r = has ? blk + (int)__ldg(M.sell_perm + rn) : blk;
  const int len = has ? (int)__ldg(M.sell_len + rn) : 0;  // not behind the permutation load
  const bool lng = has && len > kThreadRowMax;
  if (t == 0) nlr = 0;
  if (has && !lng) {
    const int rg = r + M.row_off;
    double lo = 0.0, up = 0.0;
    if (Op::SYM && M.diag) up = __ldg(M.diag + r) * o.gather(rg);
    const int64_t soff = __ldg(M.sell_off + (rn >> 5));
    for (int k = 0; k < len; k += AQP_SELL_BATCH) {
      int cc[AQP_SELL_BATCH];
      double pv[AQP_SELL_BATCH];
      sell_load<!Op::SYM>(M, soff, rn & 31, k, len, cc, pv);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u)
        if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u) {
        if (k + u < len) {
          if (Op::SYM && cc[u] < rg) lo += pv[u]; else up += pv[u];
        }
      }
    }
    ssum[r - blk] = Op::SYM ? lo + up : up;
  }
  if (__syncthreads_count(lng)) {  // rare: rows longer than a thread's share
    if (lng) lrow[atomicAdd(&nlr, 1)] = r;  // any order: each long row is summed on its own
    __syncthreads();
    const int nl = nlr;
    for (int i = 0; i < nl; ++i) {
      const int rr = lrow[i], rg = rr + M.row_off;
      RedVals<2, 0> lu;
      lu.zero();
      if (Op::SYM && M.diag && t == 0) lu.s[1] = __ldg(M.diag + rr) * o.gather(rg);
      for (int k = __ldg(M.ptr + rr) + t, ke = __ldg(M.ptr + rr + 1); k < ke; k += kThreads) {
        const int c = __ldg(M.idx + k);
        const double pv = __ldg(M.val + k) * o.gather(c);
        if (Op::SYM && c < rg) lu.s[0] += pv; else lu.s[1] += pv;
      }
      block_reduce<2, 0>(lu, sred);
      if (t == 0) ssum[rr - blk] = Op::SYM ? lu.s[0] + lu.s[1] : lu.s[1];
      __syncthreads();  // sred is reused by the next row
    }
  }
  __syncthreads();
  if (has) {
    const double val = ssum[t];
    if constexpr (RowInOf<Op>::value && RowInLateOf<Op>::value) rin = o.load_row(rn);
    if constexpr (RowInOf<Op>::value) o.row_in(rn, val, rin, acc); else o.row(rn, val, acc);
  }
}

template <class Op, bool UNIFORM = false>
__global__ void __launch_bounds__(kThreads, UNIFORM ? UniformBlocksOf<Op>::value : AQP_SPMV_MIN_BLOCKS) spmv_op(DevCsr M, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  // static matrix data first: the plan item does not depend on the predecessor
  PlanItem it;
  if (UNIFORM || M.uniform) {
    it.kind = kItemThread;
    it.row0 = blockIdx.x * kThreads;
    it.row1 = min(it.row0 + kThreads, M.rows);
  } else {
    it = M.plan[blockIdx.x];
  }
  pdl_wait();
  trace_mark(g, 0);
  if (op.skip()) return;
  Op o = op;
  o.prepare();
  // WARP-item staging buffer: dynamic, launched with M.smem_bytes (0 when the
  // matrix has no WARP items, so THREAD-only passes keep full occupancy)
  extern __shared__ double dyn_smem[];
  double *sprod = dyn_smem;
  int *scol = reinterpret_cast<int *>(dyn_smem + kTileNnz);
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<NS, NM> acc;
  acc.zero();
  spmv_item<Op, UNIFORM>(M, it, o, acc, sprod, scol, sred);
  pdl_trigger();
  if constexpr (Op::FINAL) {
    if (grid_end<NS, NM, SplitOf<Op>::value>(acc, g, sred)) o.finalize(acc);
  }
}

// a SELL-P matrix (DevCsr::sell_perm): its own instantiation, so the extra
// registers of the sorted path never touch the natural uniform kernels
template <class Op>
__global__ void __launch_bounds__(kThreads, UniformBlocksOf<Op>::value) spmv_sellp_op(DevCsr M, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  pdl_wait();
  trace_mark(g, 0);
  if (op.skip()) return;
  Op o = op;
  o.prepare();
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<NS, NM> acc;
  acc.zero();
  spmv_sellp_block<Op>(M, o, acc, sred);
  pdl_trigger();
  if constexpr (Op::FINAL) {
    if (grid_end<NS, NM, SplitOf<Op>::value>(acc, g, sred)) o.finalize(acc);
  }
}

// ---------------------------------------------------------------- banded ring path
// SpMV passes over banded matrices (C5's A, A', Q: every row's columns lie
// within +-w of the row) gather from a ring of the source vector held in
// shared memory instead of from L2.  One 1024-thread CTA per SM walks a
// contiguous strip of row groups (RT rows = RT / 256 tiles); per
// group it adds the ~RT columns the band newly reaches (DevCsr::win, read
// from HBM once per strip) while the group's rows gather their products from
// the ring -- random 8-byte L2 sector reads become shared-memory loads, and the
// matrix stream has the memory system to itself.  Each 256-thread sub-block
// runs one tile exactly as spmv_op / spmv_sellp_op would (same row -> thread
// map, same per-row summation order, same xor-shuffle + warp-order reduction,
// partials stored at the tile's block slot), so results and reductions are
// bitwise those of the non-ring kernels.  Measured on a C5-shaped pass with a
// light epilogue (scripts/native/band_bench.cu): 1.33 -> 1.05 ms.

// named barrier of sub-block `sub` (ids 1..kRingSub; 0 is __syncthreads)
__device__ __forceinline__ void sub_sync(int sub) {
  asm volatile("bar.sync %0, %1;" ::"r"(sub + 1), "r"(kThreads) : "memory");
}
__device__ __forceinline__ int sub_sync_count(int sub, bool pred) {
  int n;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.popc.u32 %0, %2, %3, p;\n\t}"
      : "=r"(n)
      : "r"((unsigned)pred), "r"(sub + 1), "r"(kThreads)
      : "memory");
  return n;
}

// block_reduce over one 256-thread sub-block (same tree, same warp order)
template <int NS, int NM>
__device__ __forceinline__ void sub_reduce(RedVals<NS, NM> &v, double *smem, int sub) {
  constexpr int NT = NS + NM;
  if constexpr (NT == 0) return;
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & (kWarps - 1);
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
  sub_sync(sub);
  if ((threadIdx.x & (kThreads - 1)) == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) v.s[i] = smem[i];
#pragma unroll
    for (int i = 0; i < NM; ++i) v.m[i] = smem[NS + i];
    for (int w = 1; w < kWarps; ++w) {
#pragma unroll
      for (int i = 0; i < NS; ++i) v.s[i] += smem[w * NT + i];
#pragma unroll
      for (int i = 0; i < NM; ++i) v.m[i] = nanmax(v.m[i], smem[w * NT + NS + i]);
    }
  }
  sub_sync(sub);
}

// the op with its gather served from the ring of S columns
template <class Op, int S>
struct RingOp : Op {
  const double *ring_;
  __device__ __forceinline__ double gather(int c) const { return ring_[(unsigned)c % S]; }
};

#ifndef AQP_RING_ROWIN_EARLY  // 1: ring rows load their epilogue operands before the row sum
#define AQP_RING_ROWIN_EARLY 1   // (C5, every op on the ring: P2 1.865 -> 1.781 ms, P1 2.429 -> 2.325)
#endif
template <class O>
struct RingLate {
  static constexpr bool value = RowInLateOf<O>::value && !AQP_RING_ROWIN_EARLY;
};

// row r of a natural SELL-32 matrix (spmv_item's THREAD path on SELL storage)
template <class O>
__device__ __forceinline__ void ring_sell_row(const DevCsr &M, const O &o, int r, RedVals<O::NS, O::NM> &acc) {
  if (r >= M.rows) return;
  using RowIn = typename RowInOf<O>::type;
  RowIn rin{};
  if constexpr (RowInOf<O>::value && !RingLate<O>::value) rin = o.load_row(r);
  const int b = __ldg(M.ptr + r), e = __ldg(M.ptr + r + 1);
  const int rg = r + M.row_off;
  double lo = 0.0, up = 0.0;
  if (O::SYM && M.diag) up = __ldg(M.diag + r) * o.gather(rg);
  const int len = e - b;
  if constexpr (!O::SYM) {
    const int64_t soff = __ldg(M.sell_off + (r >> 5));
    for (int k = 0; k < len; k += AQP_SELL_BATCH) {
      int cc[AQP_SELL_BATCH];
      double pv[AQP_SELL_BATCH];
      sell_load<true>(M, soff, r & 31, k, len, cc, pv);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u)
        if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u)
        if (k + u < len) up += pv[u];
    }
  } else {
    const int64_t base = __ldg(M.sell_off + (r >> 5)) + (r & 31);
    for (int k = 0; k < len; k += AQP_SELL_BATCH) {
      int cc[AQP_SELL_BATCH];
      double pv[AQP_SELL_BATCH];
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u) {
        const bool in = k + u < len;
        cc[u] = in ? __ldg(M.sell_idx + base + 32 * (k + u)) : 0;
        pv[u] = in ? __ldg(M.sell_val + base + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u)
        if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u) {
        if (k + u < len) {
          if (O::SYM && cc[u] < rg) lo += pv[u]; else up += pv[u];
        }
      }
    }
  }
  const double val = O::SYM ? lo + up : up;
  if constexpr (RowInOf<O>::value && RingLate<O>::value) rin = o.load_row(r);
  if constexpr (RowInOf<O>::value) o.row_in(r, val, rin, acc); else o.row(r, val, acc);
}

// tile `tile` of a SELL-P matrix on sub-block `sub` (spmv_sellp_block with
// named barriers and the sub-block's shared arrays)
template <class O>
__device__ __forceinline__ void ring_sellp_tile(const DevCsr &M, const O &o, int tile, int sub,
                                                RedVals<O::NS, O::NM> &acc, double *sred, double *ssum, int *lrow,
                                                int *nlr) {
  const int blk = tile * kThreads, t = threadIdx.x & (kThreads - 1);
  const int rn = blk + t;
  using RowIn = typename RowInOf<O>::type;
  RowIn rin{};
  const bool has = rn < M.rows;
  if constexpr (RowInOf<O>::value && !RingLate<O>::value)
    if (has) rin = o.load_row(rn);
  const int r = has ? blk + (int)__ldg(M.sell_perm + rn) : blk;
  const int len = has ? (int)__ldg(M.sell_len + rn) : 0;  // not behind the permutation load
  const bool lng = has && len > kThreadRowMax;
  if (t == 0) *nlr = 0;
  if (has && !lng) {
    const int rg = r + M.row_off;
    double lo = 0.0, up = 0.0;
    if (O::SYM && M.diag) up = __ldg(M.diag + r) * o.gather(rg);
    const int64_t soff = __ldg(M.sell_off + (rn >> 5));
    for (int k = 0; k < len; k += AQP_SELL_BATCH) {
      int cc[AQP_SELL_BATCH];
      double pv[AQP_SELL_BATCH];
      sell_load<!O::SYM>(M, soff, rn & 31, k, len, cc, pv);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u)
        if (k + u < len) pv[u] = pv[u] * o.gather(cc[u]);
#pragma unroll
      for (int u = 0; u < AQP_SELL_BATCH; ++u) {
        if (k + u < len) {
          if (O::SYM && cc[u] < rg) lo += pv[u]; else up += pv[u];
        }
      }
    }
    ssum[r - blk] = O::SYM ? lo + up : up;
  }
  if (sub_sync_count(sub, lng)) {
    if (lng) lrow[atomicAdd(nlr, 1)] = r;
    sub_sync(sub);
    const int nl = *nlr;
    for (int i = 0; i < nl; ++i) {
      const int rr = lrow[i], rg = rr + M.row_off;
      RedVals<2, 0> lu;
      lu.zero();
      if (O::SYM && M.diag && t == 0) lu.s[1] = __ldg(M.diag + rr) * o.gather(rg);
      for (int k = __ldg(M.ptr + rr) + t, ke = __ldg(M.ptr + rr + 1); k < ke; k += kThreads) {
        const int c = __ldg(M.idx + k);
        const double pv = __ldg(M.val + k) * o.gather(c);
        if (O::SYM && c < rg) lu.s[0] += pv; else lu.s[1] += pv;
      }
      sub_reduce<2, 0>(lu, sred, sub);
      if (t == 0) ssum[rr - blk] = O::SYM ? lu.s[0] + lu.s[1] : lu.s[1];
      sub_sync(sub);
    }
  }
  sub_sync(sub);
  if (has) {
    const double val = ssum[t];
    if constexpr (RowInOf<O>::value && RingLate<O>::value) rin = o.load_row(rn);
    if constexpr (RowInOf<O>::value) o.row_in(rn, val, rin, acc); else o.row(rn, val, acc);
  }
}

// Op::RING_CLASS (1: the BB gradient, 2: A'y of P1, 0: every other op)
// selects the ops AQP_RING_OFF (bit mask, default 0b110) keeps on the tile
// kernels.  Measured on C5 (bench
// kernel table, same box): the A x̄ pass P2 1.998 -> 1.863 ms and the power
// iteration gain; the BB gradient (Q's +-1000 band already hits L1/L2, seven
// epilogue streams) 1.17 -> 1.75 ms and A'y (P1, SELL-P with its per-tile
// hand-off barriers, five epilogue streams) 2.29 -> 2.43 ms lose: with one
// 1024-thread CTA per SM and a barrier per group the epilogue loads of a heavy
// op are exposed, where 48 independent warps of the tile kernel hide them.
template <class Op, class = void>
struct RingClassOf {
  static constexpr int value = 0;
};
template <class Op>
struct RingClassOf<Op, std::void_t<decltype(Op::RING_CLASS)>> {
  static constexpr int value = Op::RING_CLASS;
};
// ops the ring kernel serves: no reduction, or split reductions (partials
// only -- the last-block ticket of cold ops stays with spmv_op)
template <class Op>
constexpr bool kRingable = !Op::FINAL || SplitOf<Op>::value;

template <class Op, bool SELLP, int RT>
__global__ void __launch_bounds__(RT, kRingRT / RT) spmv_ring_op(DevCsr M, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  constexpr int kRingSub = RT / kThreads, S = ring_cols(RT);
  extern __shared__ double ring[];
  __shared__ double sred[kRingSub][kWarps * kMaxRed];
  __shared__ double ssum[SELLP ? RT : 1];
  __shared__ int lrow[SELLP ? RT : 1];
  __shared__ int nlr[kRingSub];
  pdl_wait();
  trace_mark(g, 0);
  if (op.skip()) return;
  RingOp<Op, S> o;
  static_cast<Op &>(o) = op;
  o.prepare();
  o.ring_ = ring;
  const Op &src = o;  // the vector the ring caches, through the op's own gather
  const int t = threadIdx.x, sub = t / kThreads;
  const int ng = M.win_groups;
  const int g0 = (int)((int64_t)blockIdx.x * ng / gridDim.x);
  const int g1 = (int)((int64_t)(blockIdx.x + 1) * ng / gridDim.x);
  if (g0 < g1) {
    const int2 w0 = M.win[g0];
    for (int c = w0.x + t; c <= w0.y; c += RT) ring[(unsigned)c % S] = src.gather(c);
    int have = w0.y;
    __syncthreads();
    const unsigned nb = (unsigned)M.nitems;
    for (int gi = g0; gi < g1; ++gi) {
      // the next group's new columns: loaded now, stored after this group's
      // rows (the plan guarantees win[g+1].y - win[g].x < S, so they never
      // overwrite a column this group still reads)
      const int nh = gi + 1 < g1 ? M.win[gi + 1].y : have;
      const int c0 = have + 1 + t, c1 = c0 + RT;
      const double p0 = c0 <= nh ? src.gather(c0) : 0.0;
      const double p1 = c1 <= nh ? src.gather(c1) : 0.0;
      const int tile = gi * kRingSub + sub;
      if (tile < M.nitems) {
        RedVals<NS, NM> acc;
        acc.zero();
        if constexpr (SELLP)
          ring_sellp_tile(M, o, tile, sub, acc, sred[sub], ssum + sub * kThreads, lrow + sub * kThreads, nlr + sub);
        else
          ring_sell_row(M, o, tile * kThreads + (t & (kThreads - 1)), acc);
        if constexpr (Op::FINAL && NS + NM > 0) {
          sub_reduce<NS, NM>(acc, sred[sub], sub);
          if ((t & (kThreads - 1)) == 0) {
#pragma unroll
            for (int i = 0; i < NS; ++i) g.partials[(size_t)i * nb + tile] = acc.s[i];
#pragma unroll
            for (int i = 0; i < NM; ++i) g.partials[(size_t)(NS + i) * nb + tile] = acc.m[i];
          }
        }
      }
      if (c0 <= nh) ring[(unsigned)c0 % S] = p0;
      if (c1 <= nh) ring[(unsigned)c1 % S] = p1;
      have = nh;
      __syncthreads();
    }
  }
  pdl_trigger();
}

// Op::BATCH (optional, with `struct In; In load(i) const; void elem_in(i,
// const In&, RedVals&) const`): the loads of BATCH grid-stride iterations are
// issued before any of their stores (the compiler cannot hoist them itself:
// the stores may alias), then the elements run in the same order -- the same
// elements per thread in the same order, so reductions are bitwise those of
// the plain loop.
template <class Op, class = void>
struct BatchOf {
  static constexpr int value = 0;
};
template <class Op>
struct BatchOf<Op, std::void_t<decltype(Op::BATCH)>> {
  static constexpr int value = Op::BATCH;
};

template <class Op>
__global__ void __launch_bounds__(kThreads) elem_op(int64_t n, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  pdl_wait();
  trace_mark(g, 1);
  if (op.skip()) return;
  Op o = op;
  o.prepare();
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<NS, NM> acc;
  acc.zero();
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  if constexpr (BatchOf<Op>::value > 0) {
    constexpr int U = BatchOf<Op>::value;
    for (int64_t i0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; i0 < n; i0 += U * stride) {
      typename Op::In in[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < n) in[u] = o.load(i0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < n) o.elem_in(i0 + u * stride, in[u], acc);
    }
  } else {
#pragma unroll 4
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) o.elem(i, acc);
  }
  pdl_trigger();
  if constexpr (Op::FINAL) {
    if (grid_end<NS, NM, SplitOf<Op>::value>(acc, g, sred)) o.finalize(acc);
  }
}

// the fold + finalize of a SPLIT op whose main launch had `nb` blocks
template <class Op>
__global__ void __launch_bounds__(kThreads) fin_op(Op op, GridRed g, unsigned nb) {
  constexpr int NS = Op::NS, NM = Op::NM;
  pdl_wait();
  // one block: let the next kernel's blocks get resident now -- unless this
  // block waits on peers (row shards), whose dependents must not occupy SMs
  // while it spins
  const bool shard = g.comm.nranks > 1;
  if (!shard) pdl_trigger();
  trace_mark(g, 2);
  if (op.skip()) {
    pdl_trigger();
    return;
  }
  Op o = op;
  o.prepare();
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<NS, NM> a;
  fold_partials<NS, NM>(a, g.partials, nb, sred);
  comm_allreduce<NS, NM>(a, g.comm);
  if (shard) pdl_trigger();
  if (threadIdx.x == 0) o.finalize(a);
  trace_mark(g, 3);
}

// barrier over the ranks (a zero-width exchange); one block
static __global__ void k_comm_barrier(GridRed g) {
  pdl_wait();
  RedVals<0, 0> a;
  comm_allreduce<0, 0>(a, g.comm);
  pdl_trigger();
}

// grid of an elementwise pass: a pure function of n (so reductions are
// reproducible), at most AQP_ELEM_BLOCKS_PER_SM 256-thread blocks per SM
#ifndef AQP_ELEM_BLOCKS_PER_SM
#define AQP_ELEM_BLOCKS_PER_SM 8
#endif
constexpr int kElemGridMax = 148 * AQP_ELEM_BLOCKS_PER_SM;
__host__ __device__ inline int elem_grid(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  if (b > kElemGridMax) b = kElemGridMax;
  return (int)b;
}

}  // namespace aqp
