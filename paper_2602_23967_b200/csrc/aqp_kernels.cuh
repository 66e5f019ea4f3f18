// aqp_kernels.cuh -- the two kernel skeletons every hot op of libaqp is built from.
//
//   spmv_op<Op>: one pass over a CSR matrix (A, A', the full symmetric Q or
//     P) with the op's per-row epilogue fused in and up to kMaxRed
//     deterministic grid reductions finished by the last block (which then
//     runs the op's scalar `finalize`, e.g. the BB step-size update).
//   elem_op<Op>: one fixed-grid pass over a vector index space with the
//     same reduction/finalize tail.
//
// Op concept:
//   static constexpr int NS, NM;       number of sums / NaN-propagating maxes
//   static constexpr bool SYM;         (spmv) full symmetric matrix: the row sum
//                                      is (sum of j<r entries) + (sum of j>=r),
//                                      each sequential -- bitwise the order of
//                                      _core.pyx:62-80 sym_matvec
//   static constexpr bool FINAL;       run finalize() in the last block
//   bool skip() const;                 uniform early exit (e.g. halted window)
//   void prepare();                    per-thread setup on a private copy of the
//                                      op (resolves device-side slot indices)
//   double gather(int col) const;      (spmv) source vector entry
//   void row(int r, double v, RedVals&) const;   (spmv) epilogue for row r
//   void elem(int64_t i, RedVals&) const;        (elem)
//   void finalize(const RedVals&) const;         thread 0 of the last block
#pragma once

#include "aqp_common.cuh"

namespace aqp {

template <class Op>
__global__ void __launch_bounds__(kThreads) spmv_op(DevCsr M, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  if (op.skip()) return;
  Op o = op;
  o.prepare();
  __shared__ double sprod[kTileNnz];
  __shared__ int scol[Op::SYM ? kTileNnz : 1];
  __shared__ double sred[kWarps * kMaxRed];
  const PlanItem it = M.plan[blockIdx.x];
  RedVals<NS, NM> acc;
  acc.zero();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (it.kind == kItemThread || it.kind == kItemWarp) {
    const int k0 = it.k0, k1 = it.k1;
#pragma unroll 4
    for (int k = k0 + threadIdx.x; k < k1; k += kThreads) {
      const int c = __ldg(M.idx + k);
      sprod[k - k0] = __ldg(M.val + k) * o.gather(c);
      if constexpr (Op::SYM) scol[k - k0] = c;
    }
    __syncthreads();
    if (it.kind == kItemThread) {
      const int r = it.row0 + threadIdx.x;
      if (r < it.row1) {
        const int b = __ldg(M.ptr + r) - k0, e = __ldg(M.ptr + r + 1) - k0;
        double val;
        if constexpr (Op::SYM) {
          double lo = 0.0, up = 0.0;
          for (int j = b; j < e; ++j) {
            if (scol[j] < r) lo += sprod[j]; else up += sprod[j];
          }
          val = lo + up;
        } else {
          double a = 0.0;
          for (int j = b; j < e; ++j) a += sprod[j];
          val = a;
        }
        o.row(r, val, acc);
      }
    } else {
      for (int r = it.row0 + warp; r < it.row1; r += kWarps) {
        const int b = __ldg(M.ptr + r) - k0, e = __ldg(M.ptr + r + 1) - k0;
        double lo = 0.0, up = 0.0;
        for (int j = b + lane; j < e; j += 32) {
          if (Op::SYM && scol[j] < r) lo += sprod[j]; else up += sprod[j];
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          up += __shfl_xor_sync(0xffffffffu, up, off);
          if constexpr (Op::SYM) lo += __shfl_xor_sync(0xffffffffu, lo, off);
        }
        if (lane == 0) o.row(r, Op::SYM ? lo + up : up, acc);
      }
    }
  } else if (it.kind == kItemLongSeq) {
    if (threadIdx.x == 0) {
      const int r = it.row0;
      double lo = 0.0, up = 0.0;
      for (int k = it.k0; k < it.k1; ++k) {
        const int c = __ldg(M.idx + k);
        const double p = __ldg(M.val + k) * o.gather(c);
        if (Op::SYM && c < r) lo += p; else up += p;
      }
      o.row(r, Op::SYM ? lo + up : up, acc);
    }
  } else {
    const int r = it.row0;
    RedVals<2, 0> lu;
    lu.zero();
    for (int k = it.k0 + threadIdx.x; k < it.k1; k += kThreads) {
      const int c = __ldg(M.idx + k);
      const double p = __ldg(M.val + k) * o.gather(c);
      if (Op::SYM && c < r) lu.s[0] += p; else lu.s[1] += p;
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
      }
      __syncthreads();
      if (lastseg && threadIdx.x == 0) {
        __threadfence();
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
  if constexpr (Op::FINAL) {
    if (grid_reduce<NS, NM>(acc, g, sred)) o.finalize(acc);
  }
}

template <class Op>
__global__ void __launch_bounds__(kThreads) elem_op(int64_t n, Op op, GridRed g) {
  constexpr int NS = Op::NS, NM = Op::NM;
  if (op.skip()) return;
  Op o = op;
  o.prepare();
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<NS, NM> acc;
  acc.zero();
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) o.elem(i, acc);
  if constexpr (Op::FINAL) {
    if (grid_reduce<NS, NM>(acc, g, sred)) o.finalize(acc);
  }
}


// grid of an elementwise pass: a pure function of n (so reductions are
// reproducible), at most 8 resident 256-thread blocks on each of 148 SMs
inline int elem_grid(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

}  // namespace aqp
