// h2d.cpp — large host->device copies from caller memory that may be pageable.
//
// The reference API hands the solver a dense f64 cost matrix in ordinary
// (pageable) host memory: 800 MB at n = 10k, 3.2 GB for the 20k OT config.
// A plain cudaMemcpyAsync from pageable memory is staged by the driver at
// ~10 GB/s.  Here: if the source is already page-locked it is copied
// directly; otherwise chunks are packed into two pinned bounce buffers by
// several host threads while the previous chunk's DMA runs, so the copy
// approaches the PCIe / C2C link rate instead of a single memcpy stream.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "ctx.h"

namespace otprg {

namespace {
constexpr size_t kChunk = 64ull << 20;  // bytes per bounce buffer
constexpr size_t kDirect = 32ull << 20; // below this: one plain copy
}  // namespace

cudaError_t h2d_large(otprg_ctx* ctx, void* dst, const void* src, size_t bytes) {
  cudaStream_t s = ctx->stream;
  if (bytes < kDirect) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost)
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);  // already page-locked
  cudaGetLastError();  // (clear a lookup error on plain pageable memory)
  for (int i = 0; i < 2; ++i) {
    if (!ctx->bounce[i]) {
      cudaError_t e = cudaMallocHost(&ctx->bounce[i], kChunk);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ctx->bounce_ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
  }
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nthreads = std::min(8u, hw);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  bool used[2] = {false, false};
  for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
    const size_t len = std::min(kChunk, bytes - off);
    const int k = static_cast<int>(i & 1);
    if (used[k]) {  // the DMA that last read this buffer must be done
      cudaError_t e = cudaEventSynchronize(ctx->bounce_ev[k]);
      if (e != cudaSuccess) return e;
    }
    char* buf = static_cast<char*>(ctx->bounce[k]);
    const size_t part = (len + nthreads - 1) / nthreads;
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nthreads; ++t) {
      const size_t lo = std::min(len, t * part), hi = std::min(len, lo + part);
      if (lo < hi) pool.emplace_back([=] { std::memcpy(buf + lo, in + off + lo, hi - lo); });
    }
    std::memcpy(buf, in + off, std::min(len, part));
    for (auto& th : pool) th.join();
    cudaError_t e = cudaMemcpyAsync(out + off, buf, len, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ctx->bounce_ev[k], s);
    if (e != cudaSuccess) return e;
    used[k] = true;
  }
  return cudaSuccess;
}

void release_bounce(otprg_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (ctx->bounce[i]) cudaFreeHost(ctx->bounce[i]);
    if (ctx->bounce_ev[i]) cudaEventDestroy(ctx->bounce_ev[i]);
    ctx->bounce[i] = nullptr;
    ctx->bounce_ev[i] = nullptr;
  }
}

}  // namespace otprg
