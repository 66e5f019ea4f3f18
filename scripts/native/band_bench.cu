// Standalone design probe for the banded A / A' passes of C5 (n = m = 5e7,
// 10 nonzeros per row, columns uniform in [r - 5000, r + 5000]): SELL-32 pair
// layout, one thread per row, y = A x + b.  Compares the library's schedule
// (gathers of x from L2, 6 blocks/SM) with a strip kernel that keeps a ring of
// x in shared memory: each CTA walks a contiguous strip of RT-row groups and,
// per group, adds the (~RT) new columns its band reaches, so x is read from
// HBM/L2 once per strip instead of once per nonzero.  Not part of libaqp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 band_bench.cu -o band_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int NNZ = 10, W = 5000;

__device__ __forceinline__ uint32_t hsh(uint64_t a) {
  a ^= a >> 33; a *= 0xff51afd7ed558ccdULL; a ^= a >> 33; a *= 0xc4ceb9fe1a85ec53ULL; a ^= a >> 33;
  return (uint32_t)a;
}
// pair layout, slice width NNZ: pos = 320 s + 64 (k >> 1) + 2 lane + (k & 1)
__global__ void gen(int n, int *idx, double *val) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  int c[NNZ];
  for (int k = 0; k < NNZ; ++k) {
    int64_t v = r + (int64_t)(hsh(r * 16 + k) % (2 * W + 1)) - W;
    c[k] = (int)(v < 0 ? 0 : (v > n - 1 ? n - 1 : v));
  }
  for (int i = 1; i < NNZ; ++i) for (int j = i; j > 0 && c[j - 1] > c[j]; --j) { int t = c[j]; c[j] = c[j - 1]; c[j - 1] = t; }
  const int64_t off = (r >> 5) * 32 * NNZ;
  const int lane = r & 31;
  for (int k = 0; k < NNZ; ++k) {
    const int64_t p = off + 64 * (k >> 1) + 2 * lane + (k & 1);
    idx[p] = c[k];
    val[p] = 1.0 + (hsh(r * 16 + k + 7) & 1023) * 1e-3;
  }
}
__global__ void fillx(int64_t n, double *x, double s) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = s * (double)(i % 977) - 3.0;
}
// per-group column range
__global__ void grange(int n, int rt, const int *idx, int *lo, int *hi) {
  int g = blockIdx.x;
  int mn = INT32_MAX, mx = -1;
  for (int r = g * rt + threadIdx.x; r < min(n, (g + 1) * rt); r += blockDim.x) {
    const int64_t off = ((int64_t)r >> 5) * 32 * NNZ;
    for (int k = 0; k < NNZ; ++k) {
      int c = idx[off + 64 * (k >> 1) + 2 * (r & 31) + (k & 1)];
      mn = min(mn, c); mx = max(mx, c);
    }
  }
  for (int o = 16; o; o >>= 1) { mn = min(mn, __shfl_xor_sync(~0u, mn, o)); mx = max(mx, __shfl_xor_sync(~0u, mx, o)); }
  __shared__ int smn[32], smx[32];
  if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = mn; smx[threadIdx.x >> 5] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)blockDim.x / 32; ++w) { mn = min(mn, smn[w]); mx = max(mx, smx[w]); }
    lo[g] = mn; hi[g] = mx;
  }
}

template <int B>
__device__ __forceinline__ void loadb(const int *idx, const double *val, int64_t off, int lane, int k, int (&cc)[B], double (&pv)[B]) {
#pragma unroll
  for (int h = 0; h < B / 2; ++h) {
    const int kk = k + 2 * h;
    if (kk < NNZ) {
      const int64_t q = off + 64 * (kk >> 1) + 2 * lane;
      const int2 ci = __ldg(reinterpret_cast<const int2 *>(idx + q));
      const double2 vv = __ldg(reinterpret_cast<const double2 *>(val + q));
      cc[2 * h] = ci.x; cc[2 * h + 1] = ci.y; pv[2 * h] = vv.x; pv[2 * h + 1] = vv.y;
    } else { cc[2 * h] = cc[2 * h + 1] = 0; pv[2 * h] = pv[2 * h + 1] = 0.0; }
  }
}

template <int MINB, int B>
__global__ void __launch_bounds__(256, MINB) kbase(int n, const int *idx, const double *val, const double *x,
                                                   const double *b, double *y) {
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= n) return;
  const double bb = __ldg(b + r);
  const int64_t off = ((int64_t)r >> 5) * 32 * NNZ;
  double up = 0.0;
  for (int k = 0; k < NNZ; k += B) {
    int cc[B]; double pv[B];
    loadb<B>(idx, val, off, r & 31, k, cc, pv);
#pragma unroll
    for (int u = 0; u < B; ++u) if (k + u < NNZ) pv[u] *= x[cc[u]];
#pragma unroll
    for (int u = 0; u < B; ++u) if (k + u < NNZ) up += pv[u];
  }
  y[r] = up + bb;
}

// strip kernel: CTA c walks groups [g0, g1) of RT rows; ring of S doubles
template <int RT, int S, int MINB, int B>
__global__ void __launch_bounds__(RT, MINB) kring(int n, int ng, const int *lo, const int *hi, const int *idx,
                                                  const double *val, const double *x, const double *b, double *y) {
  extern __shared__ double ring[];
  const int t = threadIdx.x;
  const int g0 = (int)((int64_t)blockIdx.x * ng / gridDim.x), g1 = (int)((int64_t)(blockIdx.x + 1) * ng / gridDim.x);
  if (g0 >= g1) return;
  for (int c = __ldg(lo + g0) + t, e = __ldg(hi + g0); c <= e; c += RT) ring[c % S] = x[c];
  int have = __ldg(hi + g0);
  __syncthreads();
  for (int g = g0; g < g1; ++g) {
    const int r = g * RT + t;
    const int nh = g + 1 < g1 ? __ldg(hi + g + 1) : have;
    const int c0 = have + 1 + t, c1 = c0 + RT;
    const double p0 = c0 <= nh ? x[c0] : 0.0, p1 = c1 <= nh ? x[c1] : 0.0;
    if (r < n) {
      const double bb = __ldg(b + r);
      const int64_t off = ((int64_t)r >> 5) * 32 * NNZ;
      double up = 0.0;
      for (int k = 0; k < NNZ; k += B) {
        int cc[B]; double pv[B];
        loadb<B>(idx, val, off, r & 31, k, cc, pv);
#pragma unroll
        for (int u = 0; u < B; ++u) if (k + u < NNZ) pv[u] *= ring[cc[u] % S];
#pragma unroll
        for (int u = 0; u < B; ++u) if (k + u < NNZ) up += pv[u];
      }
      y[r] = up + bb;
    }
    if (c0 <= nh) ring[c0 % S] = p0;
    if (c1 <= nh) ring[c1 % S] = p1;
    have = nh;
    __syncthreads();
  }
}


int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 50000000;
  const int64_t nnz = (int64_t)((n + 31) / 32) * 32 * NNZ;
  int *idx; double *val, *x, *b, *y, *y0;
  CK(cudaMalloc(&idx, nnz * 4)); CK(cudaMalloc(&val, nnz * 8));
  CK(cudaMemset(idx, 0, nnz * 4)); CK(cudaMemset(val, 0, nnz * 8));
  CK(cudaMalloc(&x, n * 8ll)); CK(cudaMalloc(&b, n * 8ll)); CK(cudaMalloc(&y, n * 8ll)); CK(cudaMalloc(&y0, n * 8ll));
  gen<<<(n + 255) / 256, 256>>>(n, idx, val);
  fillx<<<(n + 255) / 256, 256>>>(n, x, 0.01);
  fillx<<<(n + 255) / 256, 256>>>(n, b, 0.003);
  CK(cudaDeviceSynchronize());
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const double bytes = 12.0 * n * NNZ + 8.0 * n * 3;  // matrix + x + b + y
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  std::vector<double> h0(n), h1(n);
  auto report = [&](const char *name, float ms, bool check) {
    double md = 0;
    if (check) {
      CK(cudaMemcpy(h1.data(), y, n * 8ll, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) if (h1[i] != h0[i]) { md = 1; break; }
    }
    printf("%-28s %8.3f ms  %7.0f GB/s  %s\n", name, ms, bytes / (ms * 1e6), check ? (md ? "MISMATCH" : "bitwise") : "ref");
  };
#define RUNB(MINB, B) do { \
    kbase<MINB, B><<<(n + 255) / 256, 256>>>(n, idx, val, x, b, y); CK(cudaDeviceSynchronize()); \
    cudaEventRecord(e0); for (int i = 0; i < reps; ++i) kbase<MINB, B><<<(n + 255) / 256, 256>>>(n, idx, val, x, b, y); \
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); \
    report("base minb=" #MINB " B=" #B, ms / reps, true); } while (0)
  kbase<6, 4><<<(n + 255) / 256, 256>>>(n, idx, val, x, b, y);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h0.data(), y, n * 8ll, cudaMemcpyDeviceToHost));
  RUNB(6, 4); RUNB(4, 4); RUNB(6, 10); RUNB(4, 10);
#define RUNR(RT, S, MINB, B, CPS) do { \
    const int ng = (n + RT - 1) / RT; int *lo, *hi; CK(cudaMalloc(&lo, ng * 4)); CK(cudaMalloc(&hi, ng * 4)); \
    grange<<<ng, 256>>>(n, RT, idx, lo, hi); CK(cudaDeviceSynchronize()); \
    std::vector<int> hl(ng), hh(ng); CK(cudaMemcpy(hl.data(), lo, ng * 4, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(hh.data(), hi, ng * 4, cudaMemcpyDeviceToHost)); \
    for (int g = 1; g < ng; ++g) hh[g] = std::max(hh[g], hh[g - 1]); \
    for (int g = ng - 2; g >= 0; --g) hl[g] = std::min(hl[g], hl[g + 1]); \
    bool ok = true; for (int g = 0; g + 1 < ng; ++g) ok = ok && hh[g + 1] - hl[g] < S && hh[g + 1] - hh[g] <= 2 * RT; \
    CK(cudaMemcpy(lo, hl.data(), ng * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(hi, hh.data(), ng * 4, cudaMemcpyHostToDevice)); \
    auto kf = kring<RT, S, MINB, B>; CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 8)); \
    const int grid = nsm * CPS; \
    CK(cudaMemset(y, 0, n * 8ll)); \
    kf<<<grid, RT, S * 8>>>(n, ng, lo, hi, idx, val, x, b, y); CK(cudaDeviceSynchronize()); \
    cudaEventRecord(e0); for (int i = 0; i < reps; ++i) kf<<<grid, RT, S * 8>>>(n, ng, lo, hi, idx, val, x, b, y); \
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); \
    char nm[96]; snprintf(nm, 96, "ring RT=%d S=%d cps=%d B=%d%s", RT, S, CPS, B, ok ? "" : " BADPLAN"); report(nm, ms / reps, true); \
    cudaFree(lo); cudaFree(hi); } while (0)
  RUNR(1024, 16384, 1, 4, 1);
  RUNR(1024, 16384, 1, 10, 1);
  RUNR(512, 12288, 2, 4, 2);
  RUNR(512, 12288, 2, 10, 2);
  RUNR(512, 16384, 1, 10, 1);
  RUNR(256, 12288, 2, 10, 2);
  RUNR(1024, 12288, 1, 10, 2);
  RUNR(512, 12288, 2, 10, 4);
  RUNR(512, 12288, 2, 10, 8);
  return 0;
}
