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
// B200 structure: one CTA of kWarps warps per SM (grid = number of SMs) and
// the n_b * chunks_per_row (row, chunk) items of kT split into equal
// contiguous ranges, one per warp, so every SM streams the same number of
// bytes.  Each warp pulls its items through its own ring of kDepth chunk
// buffers in shared memory, filled by 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx); its lane 0 refills a stage as
// soon as the warp has read it; no cross-warp synchronisation.  A row whose
// chunks span several warps ("split row") is finished by the last of those
// warps to arrive: each piece publishes its ordered k = 0 positions (up to
// kLowCap) and its minimum, and the last arriver concatenates the pieces in
// chunk order.
#include "device_common.cuh"
#include "kernels.h"

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

// One piece of a split row (2 slots per warp: its first and its last row).
struct PropPiece {
  int32_t cnt, full_pos;
  uint32_t mn, pad;
  int32_t pos[kLowCap];
};

// Item range of warp w: [w * total / W, (w + 1) * total / W).
__device__ __forceinline__ long long item_start(long long w, long long total, long long W) {
  return w * total / W;
}
__device__ __forceinline__ long long warp_of_item(long long i, long long total, long long W) {
  long long w = i * W / total;
  while (w + 1 < W && item_start(w + 1, total, W) <= i) ++w;
  while (w > 0 && item_start(w, total, W) > i) --w;
  return w;
}

template <typename T>
__global__ void __launch_bounds__(kStreamThreads, 1)
    propose_stream_kernel(const T* __restrict__ kT, int lda, int n_b, int chunk_bytes,
                          int chunks_per_row, int4* __restrict__ lmeta,
                          unsigned long long* __restrict__ lent, T* __restrict__ rowmin,
                          PropPiece* __restrict__ pieces, int* __restrict__ row_cnt, Ctl* ctl) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);  // elements per 16-byte vector
  extern __shared__ __align__(128) unsigned char ring[];  // kWarps * kDepth * chunk_bytes
  __shared__ __align__(8) unsigned long long full_bar[kWarps][kDepth];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long W = (long long)gridDim.x * kWarps;
  const long long gw = (long long)blockIdx.x * kWarps + warp;
  const size_t row_bytes = (size_t)lda * sizeof(T);
  const long long total = (long long)n_b * chunks_per_row;
  const long long it0 = item_start(gw, total, W), it1 = item_start(gw + 1, total, W);
  const int items = (int)(it1 - it0);
  const int chunk_elems = chunk_bytes / (int)sizeof(T);
  unsigned char* my_ring = ring + (size_t)warp * kDepth * chunk_bytes;
  unsigned long long* bars = full_bar[warp];

  if (threadIdx.x == 0) atomicMin(&ctl->prop_t0, globaltimer());
  if (lane == 0) {
    for (int st = 0; st < kDepth; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto chunk_len = [&](int c) -> unsigned {
    return (unsigned)min((size_t)chunk_bytes, row_bytes - (size_t)c * chunk_bytes);
  };
  auto issue = [&](int k) {  // lane 0: load this warp's k-th item into stage k % kDepth
    const long long it = it0 + k;
    const int st = k % kDepth;
    const int b = (int)(it / chunks_per_row), c = (int)(it % chunks_per_row);
    const unsigned len = chunk_len(c);
    const char* src = reinterpret_cast<const char*>(kT) + (size_t)b * row_bytes + (size_t)c * chunk_bytes;
    mbar_expect_tx(&bars[st], len);
    bulk_g2s(my_ring + (size_t)st * chunk_bytes, src, len, &bars[st]);
  };
  if (lane == 0)
    for (int k = 0; k < min(kDepth, items); ++k) issue(k);

  int cnt = 0, full_pos = -1;
  uint32_t mn = 0xffffffffu;
  unsigned long long bytes = 0;
  int b = items ? (int)(it0 / chunks_per_row) : 0, c = items ? (int)(it0 % chunks_per_row) : 0;
  int st = 0;
  unsigned parity = 0;
  bool whole = false, first_row = true;
  int32_t* piece_pos = nullptr;
  for (int k = 0; k < items; ++k) {
    if (k == 0 || c == 0) {  // a row (piece) starts
      cnt = 0;
      full_pos = -1;
      mn = 0xffffffffu;
      whole = c == 0 && (long long)(b + 1) * chunks_per_row <= it1;
      piece_pos = pieces[2 * gw + (first_row ? 0 : 1)].pos;
    }
    mbar_wait(&bars[st], parity);
    const unsigned len = chunk_len(c);
    const int nv = (int)len / 16;
    const uint4* src = reinterpret_cast<const uint4*>(my_ring + (size_t)st * chunk_bytes);
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
            if (lane == 0) {
              if (whole) lent[(size_t)b * kLowCap + cnt] = (unsigned long long)(uint32_t)pos;  // (k=0)<<32|a
              else piece_pos[cnt] = pos;
            }
            if (cnt == kLowCap - 1) full_pos = pos;
            ++cnt;
          }
        }
      }
    }
    __syncwarp();  // the warp is done reading stage st
    if (lane == 0) {
      bytes += len;
      if (k + kDepth < items) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + kDepth);
      }
    }
    if (c == chunks_per_row - 1 || k == items - 1) {  // this warp's piece of row b ends
      const uint32_t m = __reduce_min_sync(kFull, SD::hmin(mn));
      if (whole) {
        if (lane == 0) {
          lmeta[b] = make_int4(0, full_pos >= 0 ? full_pos + 1 : lda, cnt, 0);
          rowmin[b] = (T)m;
        }
      } else {
        // split row: publish the piece; the last of the row's warps merges
        const long long ws = warp_of_item((long long)b * chunks_per_row, total, W);
        const long long we = warp_of_item((long long)(b + 1) * chunks_per_row - 1, total, W);
        int prev = 0;
        if (lane == 0) {
          PropPiece* pc = &pieces[2 * gw + (first_row ? 0 : 1)];
          pc->cnt = cnt;
          pc->mn = m;
          __threadfence();
          prev = atomicAdd(row_cnt + b, 1);
        }
        prev = __shfl_sync(kFull, prev, 0);
        if (prev == (int)(we - ws)) {
          __threadfence();
          if (lane == 0) {
            int tot = 0, fpos = -1;
            uint32_t rmin = 0xffffffffu;
            for (long long w = ws; w <= we; ++w) {
              const bool w_first = item_start(w, total, W) / chunks_per_row == b;
              const PropPiece* pc = &pieces[2 * w + (w_first ? 0 : 1)];
              const int pcnt = __ldcg(&pc->cnt);
              rmin = min(rmin, __ldcg(&pc->mn));
              for (int q = 0; q < pcnt && tot < kLowCap; ++q, ++tot) {
                const int pos = __ldcg(&pc->pos[q]);
                lent[(size_t)b * kLowCap + tot] = (unsigned long long)(uint32_t)pos;
                if (tot == kLowCap - 1) fpos = pos;
              }
            }
            lmeta[b] = make_int4(0, fpos >= 0 ? fpos + 1 : lda, tot, 0);
            rowmin[b] = (T)rmin;
            row_cnt[b] = 0;  // ready for the next launch
          }
        }
      }
      first_row = false;
    }
    if (++c == chunks_per_row) c = 0, ++b;
    if (++st == kDepth) st = 0, parity ^= 1u;
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

size_t propose_stream_scratch_bytes(int num_sms) {
  return (size_t)num_sms * kWarps * 2 * sizeof(PropPiece);
}

cudaError_t launch_propose_stream(const void* kT, int lda, int n_b, int width, int4* lmeta,
                                  unsigned long long* lent, void* rowmin, void* scratch, int* row_cnt,
                                  Ctl* ctl, int num_sms, cudaStream_t s) {
  const int chunk = propose_stream_chunk(width, lda);
  const int cpr = (lda * width + chunk - 1) / chunk;
  const size_t smem = (size_t)kWarps * kDepth * chunk;
  // one CTA per SM, equal item ranges per warp (every SM streams the same bytes)
  const int grid = num_sms;
  // raise the opt-in shared-memory limit once per device and width
  static size_t smem_set[64][3] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  size_t* smem_set_dev = smem_set[dev & 63];
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    auto fn = propose_stream_kernel<T>;
    size_t& set = smem_set_dev[sizeof(T) == 1 ? 0 : sizeof(T) == 2 ? 1 : 2];
    if (set < smem) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(set = smem));
    fn<<<grid, kStreamThreads, smem, s>>>(static_cast<const T*>(kT), lda, n_b, chunk, cpr, lmeta, lent,
                                          static_cast<T*>(rowmin), static_cast<PropPiece*>(scratch),
                                          row_cnt, ctl);
    return 0;
  });
  return cudaGetLastError();
}

}  // namespace otprg
