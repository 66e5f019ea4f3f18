// aqp_xfer.cu -- bulk host <-> device copies of the problem data and results.
//
// A solve call starts from the caller's (pageable, numpy) arrays: at C5 that is
// 13.6 GB of CSR + vectors in and 1.2 GB of x / y / slack out.  A pageable
// cudaMemcpy runs at ~10 GB/s H2D and ~4.5 GB/s D2H on the B200 box; this
// engine stages through pinned buffers instead: T host threads each own two
// pinned chunks and a stream, and pipeline memcpy(host <-> pinned) against
// the DMA of the other chunk (measured 45 GB/s H2D with 8 threads x 16-32 MB,
// scripts/h2d_probe.py).  The pinned pool is allocated once per process
// (cudaHostAlloc synchronises the device, so never per call) and reused; a
// mutex serialises transfers (one pool).
//
// Small copies (< kStagedMin) go straight through cudaMemcpy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "aqp_common.cuh"
#include "aqp_internal.h"

namespace aqp {

namespace {

constexpr int kXferThreads = 8;
constexpr size_t kXferChunk = size_t(32) << 20;  // bytes per pinned buffer (16 MB: 33 GB/s)
constexpr size_t kStagedMin = size_t(8) << 20;

struct XferPool {
  std::mutex mu;
  bool ready = false;
  void *buf[kXferThreads][2] = {};
  // per device: one stream + two events per thread (created on first use)
  struct Dev {
    bool ready = false;
    cudaStream_t st[kXferThreads] = {};
    cudaEvent_t ev[kXferThreads][2] = {};
  };
  Dev dev[64];
};

XferPool &pool() {
  static XferPool p;
  return p;
}

int pool_ready(XferPool &p, int device) {
  if (!p.ready) {  // (pinning from several threads at once measured slower: driver contention)
    for (int t = 0; t < kXferThreads; ++t)
      for (int j = 0; j < 2; ++j) AQP_CUDA(cudaHostAlloc(&p.buf[t][j], kXferChunk, cudaHostAllocPortable));
    p.ready = true;
  }
  if (device < 0 || device >= 64) return fail(AQP_EINVAL, "device id out of range");
  XferPool::Dev &d = p.dev[device];
  if (!d.ready) {
    for (int t = 0; t < kXferThreads; ++t) {
      AQP_CUDA(cudaStreamCreateWithFlags(&d.st[t], cudaStreamNonBlocking));
      for (int j = 0; j < 2; ++j) AQP_CUDA(cudaEventCreateWithFlags(&d.ev[t][j], cudaEventDisableTiming));
    }
    d.ready = true;
  }
  return AQP_OK;
}

// thread t moves chunks t, t + T, ... ; H2D: memcpy into the free pinned
// buffer, then its DMA; D2H: DMA of chunk j+1 overlaps the memcpy of chunk j
void xfer_worker(XferPool &p, int device, int t, char *dev, char *host, size_t bytes, bool h2d, int *err) {
  if (cudaSetDevice(device) != cudaSuccess) {
    *err = 1;
    return;
  }
  XferPool::Dev &d = p.dev[device];
  const size_t nch = (bytes + kXferChunk - 1) / kXferChunk;
  int j = 0;
  size_t prev = (size_t)-1;
  for (size_t c = t; c < nch; c += kXferThreads, ++j) {
    const size_t off = c * kXferChunk, len = std::min(kXferChunk, bytes - off);
    void *b = p.buf[t][j & 1];
    if (h2d) {
      if (j >= 2 && cudaEventSynchronize(d.ev[t][j & 1]) != cudaSuccess) *err = 1;
      std::memcpy(b, host + off, len);
      if (cudaMemcpyAsync(dev + off, b, len, cudaMemcpyHostToDevice, d.st[t]) != cudaSuccess) *err = 1;
      if (cudaEventRecord(d.ev[t][j & 1], d.st[t]) != cudaSuccess) *err = 1;
    } else {
      if (cudaMemcpyAsync(b, dev + off, len, cudaMemcpyDeviceToHost, d.st[t]) != cudaSuccess) *err = 1;
      if (cudaEventRecord(d.ev[t][j & 1], d.st[t]) != cudaSuccess) *err = 1;
      if (prev != (size_t)-1) {  // the previous chunk has landed in the other buffer
        const size_t poff = prev * kXferChunk, plen = std::min(kXferChunk, bytes - poff);
        if (cudaEventSynchronize(d.ev[t][(j - 1) & 1]) != cudaSuccess) *err = 1;
        std::memcpy(host + poff, p.buf[t][(j - 1) & 1], plen);
      }
      prev = c;
    }
  }
  if (!h2d && prev != (size_t)-1) {
    const size_t poff = prev * kXferChunk, plen = std::min(kXferChunk, bytes - poff);
    if (cudaEventSynchronize(d.ev[t][(j - 1) & 1]) != cudaSuccess) *err = 1;
    std::memcpy(host + poff, p.buf[t][(j - 1) & 1], plen);
  }
  if (cudaStreamSynchronize(d.st[t]) != cudaSuccess) *err = 1;
}

}  // namespace

// Allocate the pool and the device's streams now (aqp_ctx_create: runtime
// initialisation, not per solve -- the 512 MB of pinning takes ~0.25 s).
int xfer_init(int device) {
  XferPool &p = pool();
  std::lock_guard<std::mutex> lock(p.mu);
  return pool_ready(p, device);
}

// Synchronous bulk copy on `device`; the caller orders it against its own
// stream (H2D: the destination is not in use; D2H: the source is complete).
int bulk_copy(int device, void *dev, void *host, size_t bytes, bool h2d) {
  if (bytes == 0) return AQP_OK;
  if (bytes < kStagedMin) {
    AQP_CUDA(cudaMemcpy(h2d ? dev : host, h2d ? host : dev, bytes,
                        h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
    return AQP_OK;
  }
  XferPool &p = pool();
  std::lock_guard<std::mutex> lock(p.mu);
  AQP_TRY(pool_ready(p, device));
  const size_t nch = (bytes + kXferChunk - 1) / kXferChunk;
  const int nt = (int)std::min<size_t>(kXferThreads, nch);
  int errs[kXferThreads] = {};
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int t = 0; t < nt; ++t)
    th.emplace_back(xfer_worker, std::ref(p), device, t, static_cast<char *>(dev), static_cast<char *>(host), bytes,
                    h2d, &errs[t]);
  for (auto &x : th) x.join();
  for (int t = 0; t < nt; ++t)
    if (errs[t]) return fail(AQP_ECUDA, "staged host<->device copy failed");
  return AQP_OK;
}

}  // namespace aqp

using namespace aqp;

extern "C" {

int aqp_h2d(aqp_ctx *ctx, void *dev_dst, const void *host_src, size_t bytes) {
  if (!ctx || (bytes && (!dev_dst || !host_src))) return fail(AQP_EINVAL, "NULL argument");
  return bulk_copy(ctx->device, dev_dst, const_cast<void *>(host_src), bytes, true);
}

int aqp_d2h(aqp_ctx *ctx, void *host_dst, const void *dev_src, size_t bytes) {
  if (!ctx || (bytes && (!dev_src || !host_dst))) return fail(AQP_EINVAL, "NULL argument");
  AQP_CUDA(cudaStreamSynchronize(ctx->stream));  // the source is produced on the context's stream
  return bulk_copy(ctx->device, const_cast<void *>(dev_src), host_dst, bytes, false);
}

}  // extern "C"
