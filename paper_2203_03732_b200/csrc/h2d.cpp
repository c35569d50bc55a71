// h2d.cpp — large host->device copies from caller memory that may be pageable.
//
// The reference API hands the solver a dense f64 cost matrix in ordinary
// (pageable) host memory: 800 MB at n = 10k, 3.2 GB for the 20k OT config.
// A plain cudaMemcpyAsync from pageable memory is staged by the driver at
// ~10 GB/s.  Here: if the source is already page-locked it is copied
// directly; otherwise chunks are packed into two pinned bounce buffers by
// persistent host threads while the previous chunk's DMA runs, so the copy
// approaches the PCIe / C2C link rate instead of a single memcpy stream.
// (Pinning the caller's pages in place with cudaHostRegister was measured at
// ~6 GB/s for 3.2 GB on the B200 box: far slower than packing.)
#include <algorithm>
#include <atomic>
#include <cstdlib>
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
  // Persistent packers for the whole copy: chunk i may be packed once its
  // buffer's previous DMA (chunk i-2) is done (`ready`); the main thread
  // issues chunk i's DMA once every packer has finished its slice (`packed`).
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned nthreads = std::min(16u, hw);
  if (const char* env = std::getenv("OTPRG_H2D_THREADS")) nthreads = std::max(1, std::atoi(env));
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  std::atomic<size_t> ready{0};
  std::atomic<size_t> packed{0};  // slices done, over all chunks
  std::atomic<bool> stop{false};
  auto slice = [&](unsigned t, size_t i) {
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    const size_t part = (len + nthreads - 1) / nthreads;
    const size_t lo = std::min(len, t * part), hi = std::min(len, lo + part);
    if (lo < hi) std::memcpy(static_cast<char*>(ctx->bounce[i & 1]) + lo, in + off + lo, hi - lo);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      for (size_t i = 0; i < nchunks; ++i) {
        while (ready.load(std::memory_order_acquire) <= i) {
          if (stop.load(std::memory_order_relaxed)) return;
          std::this_thread::yield();
        }
        slice(t, i);
        packed.fetch_add(1, std::memory_order_acq_rel);
      }
    });
  cudaError_t err = cudaSuccess;
  for (size_t i = 0; i < nchunks && err == cudaSuccess; ++i) {
    const int k = static_cast<int>(i & 1);
    if (i >= 2) err = cudaEventSynchronize(ctx->bounce_ev[k]);  // chunk i-2's DMA read this buffer
    if (err != cudaSuccess) break;
    ready.store(i + 1, std::memory_order_release);
    slice(0, i);
    packed.fetch_add(1, std::memory_order_acq_rel);
    while (packed.load(std::memory_order_acquire) < (i + 1) * nthreads) std::this_thread::yield();
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    err = cudaMemcpyAsync(out + off, ctx->bounce[k], len, cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaEventRecord(ctx->bounce_ev[k], s);
  }
  stop.store(true);
  for (auto& th : pool) th.join();
  if (err != cudaSuccess) return err;
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
