// Stand-alone check of the row-shard mailbox exchange (aqp_common.cuh
// comm_allreduce) with P virtual ranks = P streams of ONE process on one
// device: does the bounded-spin exchange make progress when the ranks'
// kernels share the device (hardware-queue head-of-line blocking)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include comm_test.cu -o comm_test
//   CUDA_DEVICE_MAX_CONNECTIONS=32 ./comm_test P iters [graph]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2602_23967_b200/csrc/aqp_common.cuh"
using namespace aqp;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void work(double *v, int n, int rank, int it) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = v[i] * 0.5 + rank + it;
}
__global__ void xchg(Comm c, double *out, int it) {
  RedVals<2, 1> a;
  a.s[0] = c.rank + 1.0; a.s[1] = it; a.m[0] = c.rank;
  comm_allreduce<2, 1>(a, c);
  if (threadIdx.x == 0) { out[0] += a.s[0]; out[1] += a.s[1]; out[2] = a.m[0]; }
}
int main(int argc, char **argv) {
  int P = argc > 1 ? atoi(argv[1]) : 2, iters = argc > 2 ? atoi(argv[2]) : 1000;
  bool graph = argc > 3;
  std::vector<cudaStream_t> st(P);
  std::vector<char *> ws(P);
  const size_t wsb = sizeof(CommBlock) + 4096;
  const int n = 1 << 22;
  std::vector<double *> vec(P);
  for (int r = 0; r < P; ++r) {
    CK(cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking));
    CK(cudaMalloc(&ws[r], wsb));
    CK(cudaMemset(ws[r], 0, wsb));
    CK(cudaMalloc(&vec[r], n * 8));
    CK(cudaMemset(vec[r], 0, n * 8));
  }
  std::vector<Comm> cm(P);
  for (int r = 0; r < P; ++r) {
    cm[r].rank = r; cm[r].nranks = P; cm[r].cb = (CommBlock *)ws[r]; cm[r].timeout_ns = 5000000000ull;
    for (int k = 0; k < P; ++k) cm[r].delta[k] = ws[k] - ws[r];
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st[0]));
  if (!graph) {
    for (int it = 0; it < iters; ++it)
      for (int r = 0; r < P; ++r) {
        work<<<148 * 4, 256, 0, st[r]>>>(vec[r], n, r, it);
        xchg<<<1, 32, 0, st[r]>>>(cm[r], (double *)(ws[r] + sizeof(CommBlock)), it);
      }
  } else {
    std::vector<cudaGraphExec_t> ex(P);
    for (int r = 0; r < P; ++r) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st[r], cudaStreamCaptureModeThreadLocal));
      for (int it = 0; it < iters; ++it) {
        work<<<148 * 4, 256, 0, st[r]>>>(vec[r], n, r, it);
        xchg<<<1, 32, 0, st[r]>>>(cm[r], (double *)(ws[r] + sizeof(CommBlock)), it);
      }
      CK(cudaStreamEndCapture(st[r], &g));
      CK(cudaGraphInstantiate(&ex[r], g, 0));
    }
    for (int r = 0; r < P; ++r) CK(cudaGraphLaunch(ex[r], st[r]));
  }
  for (int r = 0; r < P; ++r) CK(cudaStreamSynchronize(st[r]));
  CK(cudaEventRecord(e1, st[0]));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  int bad = 0;
  for (int r = 0; r < P; ++r) {
    CommBlock cb; double out[3];
    CK(cudaMemcpy(&cb, ws[r], sizeof(cb), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out, ws[r] + sizeof(CommBlock), 24, cudaMemcpyDeviceToHost));
    const double want0 = (double)iters * P * (P + 1) / 2, want1 = (double)P * iters * (iters - 1) / 2;
    printf("rank %d epoch %llu err %llu sum0 %.0f (want %.0f) sum1 %.0f (want %.0f) max %.0f\n", r, cb.epoch, cb.err,
           out[0], want0, out[1], want1, out[2]);
    bad |= cb.err != 0 || out[0] != want0 || out[1] != want1;
  }
  printf("%s P=%d iters=%d graph=%d: %.3f ms, %.2f us/iteration\n", bad ? "FAIL" : "OK", P, iters, (int)graph, ms,
         1e3 * ms / iters);
  return bad;
}
