// propose_kernels.cu — the phase-1 propose scan as one HBM-streaming kernel.
//
// In phase 1 every b is free with Y(b) = 1 and t(a) = -Y(a) = 0 for all a
// (init_state, assignment.cpp:54-60), so b's admissible set is exactly
// {a : k(a,b) == 0} (scan_plain, assignment.cpp:65-75, target Y(b)-1 = 0).
// This kernel streams the whole B-major kT once and records, for every row:
//   * the ascending admissible positions, up to kLowCap of them (the low-set
//     cache of solve_kernels.cu at level 0, entries (k << 32) | a with k = 0),
//     and the coverage end (position after the kLowCap-th entry, or lda);
//   * the row minimum of k (+ t = 0), which lets later phases skip rows
//     that cannot have admissible edges (rowmin in solve_kernels.cu).
// The proposal chains of phase 1 then walk these lists inside the phase
// loop.  The algorithmic traffic is n_b * lda * width bytes (SURVEY §8(d):
// n_i = n in phase 1).
//
// B200 structure: one CTA of kWarps warps per SM on every SM; every warp owns
// a contiguous range of whole rows (so each row's positions are produced in
// order by one warp) and streams them through its own ring of
// kDepth chunk buffers in shared memory, filled by 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx).  The warp's lane 0 refills a
// stage as soon as the warp has read it; there is no cross-warp
// synchronisation at all.  Row chunks are sized so kWarps * kDepth chunks
// fit in shared memory (rows above the limit are split evenly).
#include "device_common.cuh"
#include "kernels.h"
#include <algorithm>

namespace otprg {

namespace {

#ifndef OTPRG_PROP_WARPS
#define OTPRG_PROP_WARPS 16
#endif
#ifndef OTPRG_PROP_DEPTH
#define OTPRG_PROP_DEPTH 3
#endif
constexpr int kWarps = OTPRG_PROP_WARPS;
constexpr int kDepth = OTPRG_PROP_DEPTH;
constexpr int kStreamThreads = kWarps * 32;
constexpr int kMaxChunk = (192 * 1024 / (kWarps * kDepth)) / 512 * 512;  // ring <= 192 KB
constexpr int kVec = 4;              // 16-byte vectors per lane per step


template <typename T>
__global__ void __launch_bounds__(kStreamThreads, 1)
    propose_stream_kernel(const T* __restrict__ kT, int lda, int n_b, int chunk_bytes,
                          int chunks_per_row, int rows_per_warp, int4* __restrict__ lmeta,
                          unsigned long long* __restrict__ lent, T* __restrict__ rowmin, Ctl* ctl) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);  // elements per 16-byte vector
  extern __shared__ __align__(128) unsigned char ring[];  // kWarps * kDepth * chunk_bytes
  __shared__ __align__(8) unsigned long long full_bar[kWarps][kDepth];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps interleaved over the SMs (warp slot `warp` of block x is global warp
  // warp * gridDim.x + x): the active warps spread evenly over every SM
  const int gw = warp * (int)gridDim.x + (int)blockIdx.x;
  const size_t row_bytes = (size_t)lda * sizeof(T);
  // contiguous, equal row ranges per warp (the last may be shorter)
  const int row0 = gw * rows_per_warp;
  const int rows = max(0, min(n_b - row0, rows_per_warp));
  const int items = rows * chunks_per_row;  // this warp's (row, chunk) pairs, in order
  const int chunk_elems = chunk_bytes / (int)sizeof(T);
  unsigned char* my_ring = ring + (size_t)warp * kDepth * chunk_bytes;
  unsigned long long* bars = full_bar[warp];

  if (threadIdx.x == 0) atomicMin(&ctl->prop_t0, globaltimer());
  if (lane == 0) {
    for (int s = 0; s < kDepth; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto chunk_len = [&](int c) -> unsigned {
    return (unsigned)min((size_t)chunk_bytes, row_bytes - (size_t)c * chunk_bytes);
  };
  auto issue = [&](int it) {  // lane 0: load item `it` into stage it % kDepth
    const int s = it % kDepth;
    const int b = row0 + it / chunks_per_row;
    const int c = it % chunks_per_row;
    const unsigned len = chunk_len(c);
    const char* src = reinterpret_cast<const char*>(kT) + (size_t)b * row_bytes + (size_t)c * chunk_bytes;
    mbar_expect_tx(&bars[s], len);
    bulk_g2s(my_ring + (size_t)s * chunk_bytes, src, len, &bars[s]);
  };
  if (lane == 0)
    for (int it = 0; it < min(kDepth, items); ++it) issue(it);

  int cnt = 0, full_pos = -1;
  uint32_t mn = 0xffffffffu;
  unsigned long long bytes = 0;
  int b = row0, c = 0, s = 0;
  unsigned parity = 0;
  for (int it = 0; it < items; ++it) {
    if (c == 0) {
      cnt = 0;
      full_pos = -1;
      mn = 0xffffffffu;
    }
    mbar_wait(&bars[s], parity);
    const unsigned len = chunk_len(c);
    const int nv = (int)len / 16;
    const uint4* src = reinterpret_cast<const uint4*>(my_ring + (size_t)s * chunk_bytes);
    const int base = c * chunk_elems;
    for (int v0 = 0; v0 < nv; v0 += 32 * kVec) {  // warp-uniform trip count
      uint4 x[kVec];
      uint32_t m4[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const int v = v0 + j * 32 + lane;
        x[j] = v < nv ? src[v] : make_uint4(~0u, ~0u, ~0u, ~0u);
        m4[j] = SD::mn(SD::mn(x[j].x, x[j].y), SD::mn(x[j].z, x[j].w));
      }
      const uint32_t mm = SD::mn(SD::mn(m4[0], m4[1]), SD::mn(m4[2], m4[3]));
      mn = SD::mn(mn, mm);
      // fast path: no zero among this step's elements (zeros are rare)
      if (!__ballot_sync(kFull, SD::eq(mm, 0u) != 0u)) continue;
      if (cnt >= kLowCap) continue;  // list full: only the minimum matters
      // Zeros are sparse even when a step has one: find the (j, lane) vectors
      // holding them from the per-vector minima, then walk those in position
      // order (j-major, lane, element) with warp-uniform scalar steps.
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        unsigned lanes = __ballot_sync(kFull, SD::eq(m4[j], 0u) != 0u);
        while (lanes && cnt < kLowCap) {
          const int src_lane = __ffs(lanes) - 1;
          lanes &= lanes - 1;
          const uint32_t z = 0u;
          const uint32_t w0 = __shfl_sync(kFull, x[j].x, src_lane), w1 = __shfl_sync(kFull, x[j].y, src_lane);
          const uint32_t w2 = __shfl_sync(kFull, x[j].z, src_lane), w3 = __shfl_sync(kFull, x[j].w, src_lane);
          uint32_t mj = SD::bits(SD::eq(w0, z)) | (SD::bits(SD::eq(w1, z)) << SD::kEpw) |
                        (SD::bits(SD::eq(w2, z)) << (2 * SD::kEpw)) |
                        (SD::bits(SD::eq(w3, z)) << (3 * SD::kEpw));
          const int e0 = base + (v0 + j * 32 + src_lane) * kEpv;
          while (mj && cnt < kLowCap) {
            const int pos = e0 + __ffs(mj) - 1;
            mj &= mj - 1;
            if (lane == 0) lent[(size_t)b * kLowCap + cnt] = (unsigned long long)(uint32_t)pos;  // (k=0)<<32|a
            if (cnt == kLowCap - 1) full_pos = pos;
            ++cnt;
          }
        }
      }
    }
    __syncwarp();  // the warp is done reading stage s
    if (lane == 0) {
      bytes += len;
      if (it + kDepth < items) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(it + kDepth);
      }
    }
    if (c == chunks_per_row - 1) {
      const uint32_t m = __reduce_min_sync(kFull, SD::hmin(mn));
      if (lane == 0) {
        lmeta[b] = make_int4(0, full_pos >= 0 ? full_pos + 1 : lda, cnt, 0);
        rowmin[b] = (T)m;
      }
    }
    if (++c == chunks_per_row) c = 0, ++b;
    if (++s == kDepth) s = 0, parity ^= 1u;
  }
  if (lane == 0) {
    if (bytes) atomicAdd(&ctl->bytes_touched, bytes);
    atomicMax(&ctl->prop_t1, globaltimer());
  }
}

}  // namespace

int propose_stream_chunk(int width, int lda) {
  const int row_bytes = lda * width;  // a multiple of 512
  const int cpr = (row_bytes + kMaxChunk - 1) / kMaxChunk;
  return ((row_bytes / 512 + cpr - 1) / cpr) * 512;  // even split, 512 B granules
}

cudaError_t launch_propose_stream(const void* kT, int lda, int n_b, int width, int4* lmeta,
                                  unsigned long long* lent, void* rowmin, Ctl* ctl, int num_sms,
                                  cudaStream_t s) {
  const int chunk = propose_stream_chunk(width, lda);
  const int cpr = (lda * width + chunk - 1) / chunk;
  const size_t smem = (size_t)kWarps * kDepth * chunk;
  // Balance: every warp gets the same number of rows (a warp's throughput
  // is set by its own ring depth, so equal shares matter more than equal
  // warps per SM).
  // Whole rows per warp, rows_per_warp = ceil(n_b / (SMs * kWarps)), and the
  // warps spread over EVERY SM: global warp `warp * grid + block`, so each SM
  // runs n_warps / grid or one more (grid = SM count).  A/B (profiles/
  // r02_prop_ab.txt): equal row counts per warp matter (a warp is bound by its
  // own ring), the SM count does not once the memory system is saturated.
  const int max_warps = num_sms * kWarps;
  const int rpw = (n_b + max_warps - 1) / max_warps;
  const int warps = (n_b + rpw - 1) / rpw;
  const int grid = std::min(num_sms, warps);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    auto fn = propose_stream_kernel<T>;
    smem_attr_raise(fn, smem);  // (only ever raised: per function and device)
    fn<<<grid, kStreamThreads, smem, s>>>(static_cast<const T*>(kT), lda, n_b, chunk, cpr, rpw, lmeta,
                                          lent, static_cast<T*>(rowmin), ctl);
    return 0;
  });
  return cudaGetLastError();
}

}  // namespace otprg
