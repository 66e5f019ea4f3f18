// standalone check of the deterministic reduction helpers on the device
#include <cstdio>
#include <vector>
#include "../../paper_2602_23967_b200/csrc/aqp_common.cuh"
#include "../../paper_2602_23967_b200/csrc/aqp_kernels.cuh"
namespace aqp { void set_error(const std::string &) {} int fail(int c, const std::string &) { return c; } }
using namespace aqp;

__global__ void k_block(const double *in, int n, double *out) {
  __shared__ double sred[kWarps * kMaxRed];
  RedVals<1, 1> acc;
  acc.zero();
  if (threadIdx.x < n) { acc.m[0] = nanmax(acc.m[0], in[threadIdx.x]); acc.s[0] += in[threadIdx.x]; }
  block_reduce<1, 1>(acc, sred);
  if (threadIdx.x == 0) { out[0] = acc.m[0]; out[1] = acc.s[0]; }
}

struct OpMax {
  static constexpr int NS = 0, NM = 1;
  static constexpr bool SYM = false, FINAL = true;
  const double *x; double *tm; double *res;
  __device__ bool skip() const { return false; }
  __device__ void prepare() {}
  __device__ double gather(int c) const { return x[c]; }
  __device__ void row(int r, double s, RedVals<0, 1> &acc) const { tm[r] = s; acc.m[0] = nanmax(acc.m[0], fabs(s)); }
  __device__ void finalize(const RedVals<0, 1> &t) const { *res = t.m[0]; }
};

int main() {
  std::vector<double> h(20);
  double vals[20] = {0., 0.159, 0., 0.092, 0.02, 0.574, 0., 2.616, 0.439, 0., 2.012, 0., 0.82, 1.511, 0., 0.064, 1.14, 0., 3.837, 0.992};
  for (int i = 0; i < 20; ++i) h[i] = vals[i];
  double *d, *o;
  cudaMalloc(&d, 8 * 64); cudaMalloc(&o, 8 * 64);
  cudaMemcpy(d, h.data(), 160, cudaMemcpyHostToDevice);
  k_block<<<1, 256>>>(d, 20, o);
  double r[2]; cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
  printf("block max %.6f (expect 3.837) sum %.6f\n", r[0], r[1]);
  // spmv: identity 20x20
  std::vector<int> ptr(21), idx(20); std::vector<double> val(20, 1.0);
  for (int i = 0; i <= 20; ++i) ptr[i] = i;
  for (int i = 0; i < 20; ++i) idx[i] = i;
  int *dp, *di; double *dv, *tm, *res, *part; unsigned *tick; PlanItem *pl;
  cudaMalloc(&dp, 84); cudaMalloc(&di, 80); cudaMalloc(&dv, 160); cudaMalloc(&tm, 160); cudaMalloc(&res, 8);
  cudaMalloc(&part, 8 * 1024); cudaMalloc(&tick, 64); cudaMemset(tick, 0, 64); cudaMalloc(&pl, sizeof(PlanItem));
  PlanItem it{}; it.row0 = 0; it.row1 = 20; it.k0 = 0; it.k1 = 20; it.kind = kItemThread;
  cudaMemcpy(pl, &it, sizeof it, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, ptr.data(), 84, cudaMemcpyHostToDevice); cudaMemcpy(di, idx.data(), 80, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), 160, cudaMemcpyHostToDevice);
  DevCsr M; M.rows = 20; M.cols = 20; M.nnz = 20; M.ptr = dp; M.idx = di; M.val = dv; M.plan = pl; M.nitems = 1;
  OpMax op{d, tm, res};
  GridRed g{part, tick};
  spmv_op<OpMax><<<1, 256>>>(M, op, g);
  cudaError_t e = cudaDeviceSynchronize();
  double rr; cudaMemcpy(&rr, res, 8, cudaMemcpyDeviceToHost);
  printf("spmv max %.6f (expect 3.837) err %s\n", rr, cudaGetErrorString(e));
  return 0;
}
