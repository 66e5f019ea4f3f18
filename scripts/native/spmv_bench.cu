// Standalone design exploration for the BB gradient pass on a C2-shaped
// matrix (n = 1e6 rows, ~5 nnz/row, random columns): which SpMV structure
// gets closest to HBM bandwidth?  Not part of libaqp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 spmv_bench.cu -o spmv_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int T = 256;

struct Vecs { const double *x, *lin, *cen, *lo, *hi, *xo, *go; double *g; double tau; };

__device__ __forceinline__ double clip(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <int NS>
__device__ void block_sum(double (&s)[NS], double *smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off; off >>= 1)
#pragma unroll
    for (int i = 0; i < NS; ++i) s[i] += __shfl_xor_sync(~0u, s[i], off);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NS; ++i) smem[warp * NS + i] = s[i];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < NS; ++i) { double a = smem[i]; for (int w = 1; w < T / 32; ++w) a += smem[w * NS + i]; s[i] = a; }
}

__device__ __forceinline__ void epi(int r, double q, const Vecs &v, double (&acc)[7]) {
  const double x = v.x[r], c = v.cen[r], l = v.lin[r];
  const double g = (q + l) + (x - c) / v.tau;
  v.g[r] = g;
  const double nr = x - clip(x - g, v.lo[r], v.hi[r]);
  acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
  const double sd = x - v.xo[r], vd = g - v.go[r];
  acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
}

// V1: current design: tile = <=256 rows / <=2048 nnz staged in smem
struct Tile { int r0, r1, k0, k1; };
__global__ void __launch_bounds__(T, 4) v1(const Tile *tiles, const int *ptr, const int *idx, const double *val,
                                           Vecs v, double *part, unsigned *ticket, int reduce) {
  __shared__ double sp[2048];
  __shared__ double sred[64];
  const Tile t = tiles[blockIdx.x];
  int cs[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) { int k = t.k0 + threadIdx.x + u * T; cs[u] = k < t.k1 ? __ldg(idx + k) : 0; }
#pragma unroll
  for (int u = 0; u < 8; ++u) { int k = t.k0 + threadIdx.x + u * T; if (k < t.k1) sp[k - t.k0] = __ldg(val + k) * __ldg(v.x + cs[u]); }
  __syncthreads();
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  int r = t.r0 + threadIdx.x;
  if (r < t.r1) {
    double a = 0; for (int j = ptr[r] - t.k0; j < ptr[r + 1] - t.k0; ++j) a += sp[j];
    epi(r, a, v, acc);
  }
  if (!reduce) return;
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// V2: CSR-scalar, ROWS rows per thread, direct global loads (L1 catches the row segments)
template <int ROWS>
__global__ void __launch_bounds__(T) v2(int n, const int *ptr, const int *idx, const double *val, Vecs v, double *part) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const int base = (blockIdx.x * T) * ROWS + threadIdx.x;
#pragma unroll
  for (int q = 0; q < ROWS; ++q) {
    const int r = base + q * T;
    if (r < n) {
      const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
      double a = 0;
      for (int k = b; k < e; ++k) a += __ldg(val + k) * __ldg(v.x + __ldg(idx + k));
      epi(r, a, v, acc);
    }
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// V3: sub-warp of L lanes per row (L = 4 or 8), coalesced-ish segment reads, shuffle sum
template <int L>
__global__ void __launch_bounds__(T) v3(int n, const int *ptr, const int *idx, const double *val, Vecs v, double *part) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const int lane = threadIdx.x % L;
  const int r = (blockIdx.x * T + threadIdx.x) / L;
  double a = 0;
  if (r < n) {
    const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    for (int k = b + lane; k < e; k += L) a += __ldg(val + k) * __ldg(v.x + __ldg(idx + k));
  }
#pragma unroll
  for (int off = L / 2; off; off >>= 1) a += __shfl_xor_sync(~0u, a, off, L);
  if (r < n && lane == 0) epi(r, a, v, acc);
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// V4: one row per thread, epilogue operands loaded first, nnz loop unrolled (loads batched)
__global__ void __launch_bounds__(T) v4(int n, const int *ptr, const int *idx, const double *val, Vecs v, double *part) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const int r = blockIdx.x * T + threadIdx.x;
  if (r < n) {
    const double x = v.x[r], c = v.cen[r], l = v.lin[r], lo = v.lo[r], hi = v.hi[r], xo = v.xo[r], go = v.go[r];
    const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    double a = 0;
    int k = b;
    for (; k + 4 <= e; k += 4) {
      const int c0 = __ldg(idx + k), c1 = __ldg(idx + k + 1), c2 = __ldg(idx + k + 2), c3 = __ldg(idx + k + 3);
      const double p0 = __ldg(val + k) * __ldg(v.x + c0), p1 = __ldg(val + k + 1) * __ldg(v.x + c1);
      const double p2 = __ldg(val + k + 2) * __ldg(v.x + c2), p3 = __ldg(val + k + 3) * __ldg(v.x + c3);
      a += p0; a += p1; a += p2; a += p3;
    }
    for (; k < e; ++k) a += __ldg(val + k) * __ldg(v.x + __ldg(idx + k));
    const double g = (a + l) + (x - c) / v.tau;
    v.g[r] = g;
    const double nr = x - clip(x - g, lo, hi);
    acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
    const double sd = x - xo, vd = g - go;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// V5: two adjacent rows per thread, 16-byte vector loads for the epilogue vectors
__global__ void __launch_bounds__(T) v5(int n, const int *ptr, const int *idx, const double *val, Vecs v, double *part) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const int r0 = 2 * (blockIdx.x * T + threadIdx.x);
  if (r0 + 1 < n) {
    const double2 x = *(const double2 *)(v.x + r0), c = *(const double2 *)(v.cen + r0), l = *(const double2 *)(v.lin + r0);
    const double2 lo = *(const double2 *)(v.lo + r0), hi = *(const double2 *)(v.hi + r0);
    const double2 xo = *(const double2 *)(v.xo + r0), go = *(const double2 *)(v.go + r0);
    const int b = __ldg(ptr + r0), m = __ldg(ptr + r0 + 1), e = __ldg(ptr + r0 + 2);
    double a0 = 0, a1 = 0;
    int k = b;
    for (; k + 4 <= m; k += 4) {
      const int c0 = __ldg(idx + k), c1 = __ldg(idx + k + 1), c2 = __ldg(idx + k + 2), c3 = __ldg(idx + k + 3);
      const double p0 = __ldg(val + k) * __ldg(v.x + c0), p1 = __ldg(val + k + 1) * __ldg(v.x + c1);
      const double p2 = __ldg(val + k + 2) * __ldg(v.x + c2), p3 = __ldg(val + k + 3) * __ldg(v.x + c3);
      a0 += p0; a0 += p1; a0 += p2; a0 += p3;
    }
    for (; k < m; ++k) a0 += __ldg(val + k) * __ldg(v.x + __ldg(idx + k));
    for (; k + 4 <= e; k += 4) {
      const int c0 = __ldg(idx + k), c1 = __ldg(idx + k + 1), c2 = __ldg(idx + k + 2), c3 = __ldg(idx + k + 3);
      const double p0 = __ldg(val + k) * __ldg(v.x + c0), p1 = __ldg(val + k + 1) * __ldg(v.x + c1);
      const double p2 = __ldg(val + k + 2) * __ldg(v.x + c2), p3 = __ldg(val + k + 3) * __ldg(v.x + c3);
      a1 += p0; a1 += p1; a1 += p2; a1 += p3;
    }
    for (; k < e; ++k) a1 += __ldg(val + k) * __ldg(v.x + __ldg(idx + k));
    double2 g;
    g.x = (a0 + l.x) + (x.x - c.x) / v.tau;
    g.y = (a1 + l.y) + (x.y - c.y) / v.tau;
    *(double2 *)(v.g + r0) = g;
    double nr = x.x - clip(x.x - g.x, lo.x, hi.x);
    acc[0] += nr * nr; acc[1] += x.x * g.x; acc[2] += l.x * x.x; acc[3] += (x.x - c.x) * c.x;
    double sd = x.x - xo.x, vd = g.x - go.x;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
    nr = x.y - clip(x.y - g.y, lo.y, hi.y);
    acc[0] += nr * nr; acc[1] += x.y * g.y; acc[2] += l.y * x.y; acc[3] += (x.y - c.y) * c.y;
    sd = x.y - xo.y; vd = g.y - go.y;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// vectorised streaming ceiling: the same 128 MB read/write with double2 / int4 loads
__global__ void stream_vec(int n, Vecs v, const double *val, const int *idx, long nnz, double *sink) {
  double a = 0;
  const long tid = blockIdx.x * (long)T + threadIdx.x, st = (long)gridDim.x * T;
  for (long i = tid; 2 * i + 1 < n; i += st) {
    const double2 p = ((const double2 *)v.x)[i], q = ((const double2 *)v.cen)[i], r = ((const double2 *)v.lin)[i];
    const double2 s = ((const double2 *)v.lo)[i], t = ((const double2 *)v.hi)[i], u = ((const double2 *)v.xo)[i];
    const double2 w = ((const double2 *)v.go)[i];
    ((double2 *)v.g)[i] = make_double2(p.x + q.x + r.x + s.x + t.x + u.x + w.x, p.y + q.y + r.y + s.y + t.y + u.y + w.y);
  }
  for (long k = tid; 4 * k + 3 < nnz; k += st) {
    const int4 c = ((const int4 *)idx)[k];
    const double2 d0 = ((const double2 *)val)[2 * k], d1 = ((const double2 *)val)[2 * k + 1];
    a += d0.x + d1.y + c.x + c.w;
  }
  if (a == 12345.678) sink[0] = a;
}

// V6: tile design, but every independent load of the tile (row pointers,
// epilogue operands, indices, values) issued up front; gathers next
__global__ void __launch_bounds__(T, 4) v6(const Tile *tiles, const int *ptr, const int *idx, const double *val,
                                           Vecs v, double *part) {
  __shared__ double sp[2048];
  __shared__ double sred[64];
  const Tile t = tiles[blockIdx.x];
  const int r = t.r0 + threadIdx.x;
  const bool own = r < t.r1;
  double x = 0, c = 0, l = 0, lo = 0, hi = 0, xo = 0, go = 0;
  int b = 0, e = 0;
  if (own) {
    b = __ldg(ptr + r) - t.k0; e = __ldg(ptr + r + 1) - t.k0;
    x = v.x[r]; c = v.cen[r]; l = v.lin[r]; lo = v.lo[r]; hi = v.hi[r]; xo = v.xo[r]; go = v.go[r];
  }
  int cs[8];
  double vs[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    int k = t.k0 + threadIdx.x + u * T;
    cs[u] = k < t.k1 ? __ldg(idx + k) : 0;
    vs[u] = k < t.k1 ? __ldg(val + k) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) { int k = t.k0 + threadIdx.x + u * T; if (k < t.k1) sp[k - t.k0] = vs[u] * __ldg(v.x + cs[u]); }
  __syncthreads();
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  if (own) {
    double a = 0; for (int j = b; j < e; ++j) a += sp[j];
    const double g = (a + l) + (x - c) / v.tau;
    v.g[r] = g;
    const double nr = x - clip(x - g, lo, hi);
    acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
    const double sd = x - xo, vd = g - go;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// ---------------------------------------------------------------- V7: persistent, TMA-pipelined
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

constexpr int kRows = 256, kNnz = 2048;
struct __align__(16) Stage {
  int idx[kNnz + 8];
  double val[kNnz + 4];
  int ptr[kRows + 12];
  double vec[7][kRows + 4];
};

struct TileCopy { int k0a, nk_bytes_i, nk_bytes_v, r0a, rp_bytes, rv_bytes; };

__device__ __forceinline__ void issue_tile(Stage &s, uint64_t *bar, const Tile &t, const int *ptr, const int *idx,
                                           const double *val, const Vecs &v) {
  const int ki = t.k0 & ~3, ke_i = (t.k1 + 3) & ~3;   // 16 B aligned int range
  const int kv = t.k0 & ~1, ke_v = (t.k1 + 1) & ~1;   // 16 B aligned double range
  const int ri = t.r0 & ~3, re_i = (t.r1 + 1 + 3) & ~3;
  const int rv = t.r0 & ~1, re_v = (t.r1 + 1) & ~1;
  const unsigned bi = (ke_i - ki) * 4, bv = (ke_v - kv) * 8, bp = (re_i - ri) * 4, bw = (re_v - rv) * 8;
  mbar_expect_tx(bar, bi + bv + bp + 7 * bw);
  if (bi) tma_load_1d(s.idx, idx + ki, bi, bar);
  if (bv) tma_load_1d(s.val, val + kv, bv, bar);
  tma_load_1d(s.ptr, ptr + ri, bp, bar);
  const double *src[7] = {v.x, v.cen, v.lin, v.lo, v.hi, v.xo, v.go};
#pragma unroll
  for (int j = 0; j < 7; ++j) tma_load_1d(s.vec[j], src[j] + rv, bw, bar);
}

__global__ void __launch_bounds__(T, 2) v7(int ntiles, const Tile *tiles, const int *ptr, const int *idx,
                                           const double *val, Vecs v, double *part) {
  extern __shared__ __align__(16) unsigned char dyn[];
  Stage *st = reinterpret_cast<Stage *>(dyn);
  __shared__ uint64_t bars[2];
  __shared__ double sred[64];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  int it = 0;
  int t = blockIdx.x;
  if (threadIdx.x == 0 && t < ntiles) issue_tile(st[0], &bars[0], tiles[t], ptr, idx, val, v);
  for (; t < ntiles; t += gridDim.x, ++it) {
    const int b = it & 1;
    const int tn = t + gridDim.x;
    if (threadIdx.x == 0 && tn < ntiles) issue_tile(st[b ^ 1], &bars[b ^ 1], tiles[tn], ptr, idx, val, v);
    const Tile tl = tiles[t];
    mbar_wait(&bars[b], (it >> 1) & 1);
    Stage &s = st[b];
    const int oi = tl.k0 - (tl.k0 & ~3), ov = tl.k0 - (tl.k0 & ~1);
    const int nk = tl.k1 - tl.k0;
#pragma unroll
    for (int u = 0; u < kNnz / T; ++u) {
      const int k = threadIdx.x + u * T;
      if (k < nk) s.val[ov + k] = s.val[ov + k] * __ldg(v.x + s.idx[oi + k]);
    }
    __syncthreads();
    const int r = tl.r0 + threadIdx.x;
    if (r < tl.r1) {
      const int op = tl.r0 - (tl.r0 & ~3), ow = tl.r0 - (tl.r0 & ~1);
      const int j = threadIdx.x;
      const int bb = s.ptr[op + j] - tl.k0, ee = s.ptr[op + j + 1] - tl.k0;
      double a = 0;
      for (int q = bb; q < ee; ++q) a += s.val[ov + q];
      const double x = s.vec[0][ow + j], c = s.vec[1][ow + j], l = s.vec[2][ow + j], lo = s.vec[3][ow + j];
      const double hi = s.vec[4][ow + j], xo = s.vec[5][ow + j], go = s.vec[6][ow + j];
      const double g = (a + l) + (x - c) / v.tau;
      v.g[r] = g;
      const double nr = x - clip(x - g, lo, hi);
      acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
      const double sd = x - xo, vd = g - go;
      acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
    }
    __syncthreads();
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
}

// V9: thread per row, direct loads, optional separate diagonal (DIAG: the CSR
// holds off-diagonals only and d[r] * x[r] is the first term of the upper
// part -- the same summation order as the full row), last-block grid reduce
template <bool DIAG, bool TICKET>
__global__ void __launch_bounds__(T) v9(int n, const int *ptr, const int *idx, const double *val, const double *dq,
                                        Vecs v, double *part, unsigned *ticket, double *out) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  __shared__ bool last;
  const int r = blockIdx.x * T + threadIdx.x;
  if (r < n) {
    const double x = v.x[r], c = v.cen[r], l = v.lin[r], lo = v.lo[r], hi = v.hi[r], xo = v.xo[r], go = v.go[r];
    const double d = DIAG ? dq[r] : 0.0;
    const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    double lo_s = 0.0, up_s = 0.0;
    bool in_up = false;
    if (DIAG) {
      for (int k = b; k < e; ++k) {
        const int col = __ldg(idx + k);
        const double p = __ldg(val + k) * __ldg(v.x + col);
        if (col < r) lo_s += p;
        else {
          if (!in_up) { up_s = 0.0 + d * x; in_up = true; }
          up_s += p;
        }
      }
      if (!in_up) up_s = 0.0 + d * x;
    } else {
      for (int k = b; k < e; ++k) {
        const int col = __ldg(idx + k);
        const double p = __ldg(val + k) * __ldg(v.x + col);
        if (col < r) lo_s += p; else up_s += p;
      }
    }
    const double a = lo_s + up_s;
    const double g = (a + l) + (x - c) / v.tau;
    v.g[r] = g;
    const double nr = x - clip(x - g, lo, hi);
    acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
    const double sd = x - xo, vd = g - go;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (!TICKET) {
    if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (unsigned bb = threadIdx.x; bb < gridDim.x; bb += T)
    for (int i = 0; i < 7; ++i) s[i] += __ldcg(part + bb * 7 + i);
  block_sum<7>(s, sred);
  if (threadIdx.x == 0) { for (int i = 0; i < 7; ++i) out[i] = s[i]; *ticket = 0; }
}

// V10: v9 body, ticket via a release/acquire atomic (no SC fence); only warp 0
// waits for the ticket, the other warps retire immediately; the last block's
// warp 0 folds the partials
__global__ void __launch_bounds__(T) v10(int n, const int *ptr, const int *idx, const double *val, Vecs v,
                                         double *part, unsigned *ticket, double *out) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const int r = blockIdx.x * T + threadIdx.x;
  if (r < n) {
    const double x = v.x[r], c = v.cen[r], l = v.lin[r], lo = v.lo[r], hi = v.hi[r], xo = v.xo[r], go = v.go[r];
    const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    double lo_s = 0.0, up_s = 0.0;
    for (int k = b; k < e; ++k) {
      const int col = __ldg(idx + k);
      const double p = __ldg(val + k) * __ldg(v.x + col);
      if (col < r) lo_s += p; else up_s += p;
    }
    const double a = lo_s + up_s;
    const double g = (a + l) + (x - c) / v.tau;
    v.g[r] = g;
    const double nr = x - clip(x - g, lo, hi);
    acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
    const double sd = x - xo, vd = g - go;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x >= 32) return;
  unsigned tk = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 7; ++i) part[blockIdx.x * 7 + i] = acc[i];
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    tk = old;
  }
  tk = __shfl_sync(~0u, tk, 0);
  if (tk != gridDim.x - 1) return;
  // warp 0 of the last block: fold (acquire above orders the loads)
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (unsigned bb = threadIdx.x; bb < gridDim.x; bb += 32)
    for (int i = 0; i < 7; ++i) s[i] += __ldcg(part + bb * 7 + i);
#pragma unroll
  for (int off = 16; off; off >>= 1)
    for (int i = 0; i < 7; ++i) s[i] += __shfl_xor_sync(~0u, s[i], off);
  if (threadIdx.x == 0) { for (int i = 0; i < 7; ++i) out[i] = s[i]; *ticket = 0; }
}

__global__ void fin(int nb, const double *part, double *out) {
  __shared__ double sred[64];
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int bb = threadIdx.x; bb < nb; bb += T)
    for (int i = 0; i < 7; ++i) s[i] += part[bb * 7 + i];
  block_sum<7>(s, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) out[i] = s[i];
}

// V11: one wave of persistent blocks striding over row tiles; thread per row,
// direct loads; partials stored [slot][block] (coalesced fold); ticket by
// thread 0 with an SC fence, once per block
__global__ void __launch_bounds__(T) v11(int ntiles, const Tile *tiles, const int *ptr, const int *idx,
                                         const double *val, Vecs v, double *part, unsigned *ticket, double *out) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  __shared__ bool last;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const int r = tl.r0 + threadIdx.x;
    if (r < tl.r1) {
      const double x = v.x[r], c = v.cen[r], l = v.lin[r], lo = v.lo[r], hi = v.hi[r], xo = v.xo[r], go = v.go[r];
      const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
      double lo_s = 0.0, up_s = 0.0;
      for (int k = b; k < e; ++k) {
        const int col = __ldg(idx + k);
        const double p = __ldg(val + k) * __ldg(v.x + col);
        if (col < r) lo_s += p; else up_s += p;
      }
      const double a = lo_s + up_s;
      const double g = (a + l) + (x - c) / v.tau;
      v.g[r] = g;
      const double nr = x - clip(x - g, lo, hi);
      acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
      const double sd = x - xo, vd = g - go;
      acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
    }
  }
  block_sum<7>(acc, sred);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 7; ++i) part[i * nb + blockIdx.x] = acc[i];
    __threadfence();
    last = atomicAdd(ticket, 1u) == (unsigned)nb - 1;
    if (last) __threadfence();
  }
  __syncthreads();
  if (!last) return;
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  constexpr int U = 8;
  for (int b0 = threadIdx.x; b0 < nb; b0 += U * T) {
    double tmp[U][7];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 7; ++i) tmp[u][i] = (b0 + u * T < nb) ? __ldcg(part + i * nb + b0 + u * T) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 7; ++i) s[i] += tmp[u][i];
  }
  block_sum<7>(s, sred);
  if (threadIdx.x == 0) { for (int i = 0; i < 7; ++i) out[i] = s[i]; *ticket = 0; }
}

// V12: v9 body (no ticket) but every pointer comes from a slot index read from
// global memory first (the library's rotating BB buffers)
struct Slots { int xt, xo, go, g; };
__global__ void __launch_bounds__(T) v12(int n, const int *ptr, const int *idx, const double *val, const double *bufs,
                                         const Slots *slots, Vecs v, double *part) {
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};
  __shared__ double sred[64];
  const Slots sl = *slots;
  const double *xt = bufs + (long)sl.xt * n, *xo = bufs + (long)sl.xo * n, *go = bufs + (long)sl.go * n;
  double *gt = const_cast<double *>(bufs) + (long)sl.g * n;
  const int r = blockIdx.x * T + threadIdx.x;
  if (r < n) {
    const double x = xt[r], c = v.cen[r], l = v.lin[r], lo = v.lo[r], hi = v.hi[r], xov = xo[r], gov = go[r];
    const int b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    double lo_s = 0.0, up_s = 0.0;
    for (int k = b; k < e; ++k) {
      const int col = __ldg(idx + k);
      const double p = __ldg(val + k) * __ldg(xt + col);
      if (col < r) lo_s += p; else up_s += p;
    }
    const double a = lo_s + up_s;
    const double g = (a + l) + (x - c) / v.tau;
    gt[r] = g;
    const double nr = x - clip(x - g, lo, hi);
    acc[0] += nr * nr; acc[1] += x * g; acc[2] += l * x; acc[3] += (x - c) * c;
    const double sd = x - xov, vd = g - gov;
    acc[4] += sd * vd; acc[5] += sd * sd; acc[6] += vd * vd;
  }
  block_sum<7>(acc, sred);
  if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) part[i * gridDim.x + blockIdx.x] = acc[i];
}

// fold probes: 7 x nb partials stored [slot][block]
template <int TH, int MODE>
__global__ void __launch_bounds__(TH) fold_probe(int nb, const double *part, double *out) {
  double s[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < nb; b += TH)
#pragma unroll
    for (int i = 0; i < 7; ++i) s[i] += MODE ? __ldcg(part + (long)i * nb + b) : part[(long)i * nb + b];
  __shared__ double sm[TH / 32][7];
#pragma unroll
  for (int off = 16; off; off >>= 1)
#pragma unroll
    for (int i = 0; i < 7; ++i) s[i] += __shfl_xor_sync(~0u, s[i], off);
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < 7; ++i) sm[threadIdx.x >> 5][i] = s[i];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 7; ++i) { double a = 0; for (int w = 0; w < TH / 32; ++w) a += sm[w][i]; out[i] = a; }
}

// gather-only probes: sum_k val[k] * x[idx[k]] with different cache operators (MODE 0 ldg, 1 ldcg, 2 plain)
template <int MODE>
__global__ void gather_only(long nnz, const int *idx, const double *val, const double *x, double *sink) {
  double a = 0;
  const long st = (long)gridDim.x * T;
  long k = blockIdx.x * (long)T + threadIdx.x;
#pragma unroll 4
  for (; k < nnz; k += st) {
    const int c = __ldg(idx + k);
    double xv;
    if (MODE == 0) xv = __ldg(x + c);
    else if (MODE == 1) xv = __ldcg(x + c);
    else xv = x[c];
    a += __ldg(val + k) * xv;
  }
  if (a == 12345.678) sink[0] = a;
}
__global__ void idx_only(long nnz, const int *idx, const double *val, double *sink) {
  double a = 0;
  const long st = (long)gridDim.x * T;
#pragma unroll 4
  for (long k = blockIdx.x * (long)T + threadIdx.x; k < nnz; k += st) a += __ldg(val + k) * __ldg(idx + k);
  if (a == 12345.678) sink[0] = a;
}

// plain streaming reference: read 7 vectors + write 1 (64 B/row), and a copy of Q arrays
__global__ void stream_ref(int n, Vecs v, const double *val, const int *idx, long nnz, double *sink) {
  double a = 0;
  for (long i = blockIdx.x * (long)T + threadIdx.x; i < n; i += (long)gridDim.x * T) {
    a += v.x[i] + v.cen[i] + v.lin[i] + v.lo[i] + v.hi[i] + v.xo[i] + v.go[i];
    v.g[i] = a;
  }
  for (long k = blockIdx.x * (long)T + threadIdx.x; k < nnz; k += (long)gridDim.x * T) a += val[k] + idx[k];
  if (a == 12345.678) sink[0] = a;
}

__global__ void flush_read(const double2 *p, long n2, double *sink) {
  double a = 0;
  for (long i = blockIdx.x * (long)T + threadIdx.x; i < n2; i += (long)gridDim.x * T) { double2 q = __ldcs(p + i); a += q.x + q.y; }
  if (a == 1.2345) sink[0] = a;
}

int main(int argc, char **argv) {
  const int n = 1000000, per = 4;
  std::mt19937_64 rng(1);
  std::vector<int> ptr(n + 1), idx;
  std::vector<double> val;
  idx.reserve(n * 5);
  for (int i = 0; i < n; ++i) {
    ptr[i] = (int)idx.size();
    std::vector<int> cols{i};
    int extra = per + (int)(rng() % 3) - 1;  // 3..5 off-diagonals
    for (int k = 0; k < extra; ++k) cols.push_back((int)(rng() % n));
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    for (int c : cols) { idx.push_back(c); val.push_back(1.0 + (rng() % 100) * 0.01); }
  }
  ptr[n] = (int)idx.size();
  const long nnz = idx.size();
  printf("n=%d nnz=%ld (%.2f/row)\n", n, nnz, (double)nnz / n);
  std::vector<Tile> tiles;
  for (int i = 0; i < n;) {
    int s = i, kk = 0;
    while (i < n && i - s < T && kk + (ptr[i + 1] - ptr[i]) <= 2048) { kk += ptr[i + 1] - ptr[i]; ++i; }
    tiles.push_back({s, i, ptr[s], ptr[i]});
  }
  int *dptr, *didx; double *dval; Tile *dt;
  CK(cudaMalloc(&dptr, (n + 1) * 4)); CK(cudaMalloc(&didx, nnz * 4)); CK(cudaMalloc(&dval, nnz * 8));
  CK(cudaMalloc(&dt, tiles.size() * sizeof(Tile)));
  CK(cudaMemcpy(dptr, ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, idx.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dval, val.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  double *vecs; CK(cudaMalloc(&vecs, 8L * n * 8)); CK(cudaMemset(vecs, 0, 8L * n * 8));
  Vecs v{vecs, vecs + n, vecs + 2L * n, vecs + 3L * n, vecs + 4L * n, vecs + 5L * n, vecs + 6L * n, vecs + 7L * n, 0.5};
  double *part; unsigned *tk; CK(cudaMalloc(&part, 8 << 20)); CK(cudaMalloc(&tk, 64));
  char *flush; const size_t fb = 512 << 20; CK(cudaMalloc(&flush, fb)); CK(cudaMemset(flush, 0, fb));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 12.0 * nnz + 4.0 * (n + 1) + 64.0 * n;
  auto timeit = [&](const char *name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    double tot = 0; const int R = 20;
    for (int r = 0; r < R; ++r) {
      flush_read<<<148 * 8, T>>>((const double2 *)flush, (long)(fb / 16), part);
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
    }
    CK(cudaGetLastError());
    double us = tot / R * 1e3;
    printf("%-28s %8.2f us  %7.0f GB/s (alg %0.0f MB)\n", name, us, bytes / us / 1e3, bytes / 1e6);
  };
  const int nt = (int)tiles.size();
  timeit("stream_ref (64n+12nnz)", [&] { stream_ref<<<148 * 8, T>>>(n, v, dval, didx, nnz, part); });
  timeit("v1 tile+reduce", [&] { v1<<<nt, T>>>(dt, dptr, didx, dval, v, part, tk, 1); });
  timeit("v1 tile no-reduce", [&] { v1<<<nt, T>>>(dt, dptr, didx, dval, v, part, tk, 0); });
  timeit("v2 scalar 1 row/thr", [&] { v2<1><<<(n + T - 1) / T, T>>>(n, dptr, didx, dval, v, part); });
  timeit("v2 scalar 2 rows/thr", [&] { v2<2><<<(n + 2 * T - 1) / (2 * T), T>>>(n, dptr, didx, dval, v, part); });
  timeit("v2 scalar 4 rows/thr", [&] { v2<4><<<(n + 4 * T - 1) / (4 * T), T>>>(n, dptr, didx, dval, v, part); });
  timeit("idx+val only (60 MB)", [&] { idx_only<<<148 * 16, T>>>(nnz, didx, dval, part); });
  timeit("gather ldg", [&] { gather_only<0><<<148 * 16, T>>>(nnz, didx, dval, vecs, part); });
  timeit("gather ldcg", [&] { gather_only<1><<<148 * 16, T>>>(nnz, didx, dval, vecs, part); });
  timeit("gather plain", [&] { gather_only<2><<<148 * 16, T>>>(nnz, didx, dval, vecs, part); });
  timeit("v6 tile all-loads-first", [&] { v6<<<nt, T>>>(dt, dptr, didx, dval, v, part); });
  {
    // off-diagonal CSR + diagonal vector
    std::vector<int> p2(n + 1), i2; std::vector<double> v2v, dv(n, 0.0);
    for (int i = 0; i < n; ++i) {
      p2[i] = (int)i2.size();
      for (int k = ptr[i]; k < ptr[i + 1]; ++k) { if (idx[k] == i) dv[i] = val[k]; else { i2.push_back(idx[k]); v2v.push_back(val[k]); } }
    }
    p2[n] = (int)i2.size();
    int *dp2, *di2; double *dv2, *dd, *outv;
    CK(cudaMalloc(&dp2, (n + 1) * 4)); CK(cudaMalloc(&di2, i2.size() * 4)); CK(cudaMalloc(&dv2, v2v.size() * 8));
    CK(cudaMalloc(&dd, n * 8)); CK(cudaMalloc(&outv, 64));
    CK(cudaMemcpy(dp2, p2.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(di2, i2.data(), i2.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dv2, v2v.data(), v2v.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dd, dv.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(tk, 0, 64));
    const int gb = (n + T - 1) / T;
    std::vector<double> ga(n), gb2(n);
    v9<false, true><<<gb, T>>>(n, dptr, didx, dval, dd, v, part, tk, outv);
    CK(cudaMemcpy(ga.data(), v.g, n * 8, cudaMemcpyDeviceToHost));
    v9<true, true><<<gb, T>>>(n, dp2, di2, dv2, dd, v, part, tk, outv);
    CK(cudaMemcpy(gb2.data(), v.g, n * 8, cudaMemcpyDeviceToHost));
    bool same = true; for (int i = 0; i < n; ++i) same &= (ga[i] == gb2[i]);
    printf("v9 diag-split bitwise equal to full-row: %d\n", (int)same);
    timeit("v9 row/thr + ticket", [&] { v9<false, true><<<gb, T>>>(n, dptr, didx, dval, dd, v, part, tk, outv); });
    timeit("v9 row/thr no ticket", [&] { v9<false, false><<<gb, T>>>(n, dptr, didx, dval, dd, v, part, tk, outv); });
    timeit("v9 diag-split + ticket", [&] { v9<true, true><<<gb, T>>>(n, dp2, di2, dv2, dd, v, part, tk, outv); });
    {
      double *bufs; Slots *dsl; Slots hs{1, 2, 3, 4};
      CK(cudaMalloc(&bufs, 5L * n * 8)); CK(cudaMemset(bufs, 0, 5L * n * 8)); CK(cudaMalloc(&dsl, sizeof(Slots)));
      CK(cudaMemcpy(dsl, &hs, sizeof hs, cudaMemcpyHostToDevice));
      timeit("v12 slot-indirect pointers", [&] { v12<<<gb, T>>>(n, dptr, didx, dval, bufs, dsl, v, part); });
      timeit("v9 row/thr no ticket (again)", [&] { v9<false, false><<<gb, T>>>(n, dptr, didx, dval, dd, v, part, tk, outv); });
    }
    {
      const int nbp = 3907;
      timeit("fold 256 plain", [&] { fold_probe<256, 0><<<1, 256>>>(nbp, part, outv); });
      timeit("fold 256 cg", [&] { fold_probe<256, 1><<<1, 256>>>(nbp, part, outv); });
      timeit("fold 1024 plain", [&] { fold_probe<1024, 0><<<1, 1024>>>(nbp, part, outv); });
      timeit("empty-ish 1 block", [&] { fold_probe<256, 0><<<1, 256>>>(1, part, outv); });
    }
    for (int bps : {2, 4, 6, 8}) {
      char nm[64];
      snprintf(nm, sizeof nm, "v11 one-wave x%d/SM", bps);
      timeit(nm, [&] { v11<<<148 * bps, T>>>(nt, dt, dptr, didx, dval, v, part, tk, outv); });
    }
    timeit("v10 acq_rel ticket, warp0", [&] { v10<<<gb, T>>>(n, dptr, didx, dval, v, part, tk, outv); });
    timeit("v9 no ticket + fin kernel", [&] {
      v9<false, false><<<gb, T>>>(n, dptr, didx, dval, dd, v, part, tk, outv);
      fin<<<1, T>>>(gb, part, outv);
    });
  }
  {
    const int smem = 2 * sizeof(Stage);
    CK(cudaFuncSetAttribute(v7, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // correctness vs v2 on g
    v2<1><<<(n + T - 1) / T, T>>>(n, dptr, didx, dval, v, part);
    std::vector<double> g1(n), g2(n);
    // make x non-trivial
    std::vector<double> xs(n); for (int i = 0; i < n; ++i) xs[i] = (i % 97) * 0.01 - 0.3;
    CK(cudaMemcpy(vecs, xs.data(), n * 8, cudaMemcpyHostToDevice));
    v2<1><<<(n + T - 1) / T, T>>>(n, dptr, didx, dval, v, part);
    CK(cudaMemcpy(g1.data(), v.g, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(v.g, 0, n * 8));
    v7<<<148 * 2, T, smem>>>(nt, dt, dptr, didx, dval, v, part);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(g2.data(), v.g, n * 8, cudaMemcpyDeviceToHost));
    double md = 0; for (int i = 0; i < n; ++i) md = std::max(md, std::abs(g1[i] - g2[i]));
    printf("v7 vs v2 max |dg| = %g (smem %d B)\n", md, smem);
    timeit("v7 persistent TMA x2/SM", [&] { v7<<<148 * 2, T, smem>>>(nt, dt, dptr, didx, dval, v, part); });
  }
  timeit("stream_vec (double2/int4)", [&] { stream_vec<<<148 * 8, T>>>(n, v, dval, didx, nnz, part); });
  timeit("v4 row/thr prefetch+unroll", [&] { v4<<<(n + T - 1) / T, T>>>(n, dptr, didx, dval, v, part); });
  timeit("v5 2rows/thr double2", [&] { v5<<<(n / 2 + T - 1) / T, T>>>(n, dptr, didx, dval, v, part); });
  timeit("v3 subwarp 2", [&] { v3<2><<<(int)((2L * n + T - 1) / T), T>>>(n, dptr, didx, dval, v, part); });
  timeit("v3 subwarp 4", [&] { v3<4><<<(int)((4L * n + T - 1) / T), T>>>(n, dptr, didx, dval, v, part); });
  timeit("v3 subwarp 8", [&] { v3<8><<<(int)((8L * n + T - 1) / T), T>>>(n, dptr, didx, dval, v, part); });
  return 0;
}
