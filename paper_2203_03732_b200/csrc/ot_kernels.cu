// ot_kernels.cu — device side of the OT copy/cluster solver
// (reference: solve_copy_matching, src/ot.cpp:418-637).
//
// Every demand vertex a carries at most two dual clusters (ot.hpp:65-96);
// t0[a] / t1[a] = -y of its clusters in descending-y order (type max when
// absent).  For each free supply vertex b with free-copy dual y_b, the
// admissible clusters are those with y(a,ci) == k(a,b) + 1 - y_b
// (ot.cpp:488-490), i.e. k(a,b) + t_ci(a) == y_b - 1.  ot_scan_kernel streams
// row b of kT (one warp per request, 128-bit loads, packed SIMD compares
// against both cluster arrays) and returns the first K admissible (a, ci) in
// ascending a from a start position, plus where to resume if the list was
// truncated.  The serial claim step that consumes these lists runs on the
// host (ot_host.cpp).
#include <climits>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) ot_scan_kernel(const T* __restrict__ kT, int lda,
                                                      const T* __restrict__ t0,
                                                      const T* __restrict__ t1,
                                                      const int4* __restrict__ req, int nreq,
                                                      int K, int32_t* __restrict__ out,
                                                      int2* __restrict__ meta) {
  using S = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  constexpr int kU = 4;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nreq) return;
  const int4 r = req[w];  // (b, target, start, -)
  const int b = r.x;
  const uint32_t tg = S::rep((uint32_t)r.y);
  const int start = r.z;
  const uint4* rv = reinterpret_cast<const uint4*>(kT + (size_t)b * lda);
  const uint4* v0 = reinterpret_cast<const uint4*>(t0);
  const uint4* v1 = reinterpret_cast<const uint4*>(t1);
  const int nv = lda / kEpv;
  int32_t* o = out + (size_t)w * K;
  int cnt = 0, resume = -1;
  for (int v = (start / kEpv) & ~31; v < nv && resume < 0; v += 32 * kU) {
    uint4 kr[kU], a0[kU], a1[kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int vi = v + j * 32 + lane;
      if (vi < nv) {
        kr[j] = __ldg(rv + vi);
        a0[j] = __ldg(v0 + vi);
        a1[j] = __ldg(v1 + vi);
      } else {
        kr[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
        a0[j] = a1[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      if (resume >= 0) break;
      const int e0 = (v + j * 32 + lane) * kEpv;
      const uint32_t kw[4] = {kr[j].x, kr[j].y, kr[j].z, kr[j].w};
      const uint32_t w0[4] = {a0[j].x, a0[j].y, a0[j].z, a0[j].w};
      const uint32_t w1[4] = {a1[j].x, a1[j].y, a1[j].z, a1[j].w};
      uint32_t m0 = 0, m1 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        m0 |= S::bits(S::eq(S::add(kw[q], w0[q]), tg)) << (q * S::kEpw);
        m1 |= S::bits(S::eq(S::add(kw[q], w1[q]), tg)) << (q * S::kEpw);
      }
      uint32_t m = m0 | m1;
      if (e0 < start) {
        const int drop = start - e0;
        m = drop >= kEpv ? 0u : (m & (~0u << drop));
      }
      if (!__ballot_sync(kFull, m != 0)) continue;
      const int c = __popc(m);
      int inc = c;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, s);
        if (lane >= s) inc += y;
      }
      const int tot = __shfl_sync(kFull, inc, 31);
      int idx = cnt + inc - c;
      int last = -1;
      uint32_t bm = m;
      while (bm) {
        const int i = __ffs(bm) - 1;
        bm &= bm - 1;
        if (idx < K) {
          // the lower-index cluster wins when both match (they cannot: the
          // two duals differ); ci = 0 when cluster 0 matches
          o[idx] = (e0 + i) * 2 + ((m0 >> i) & 1u ? 0 : 1);
          if (idx == K - 1) last = e0 + i;
        }
        ++idx;
      }
      if (cnt + tot >= K) {
        const unsigned src = __ballot_sync(kFull, last >= 0);
        resume = __shfl_sync(kFull, last, __ffs(src) - 1) + 1;
        cnt = K;
      } else {
        cnt += tot;
      }
    }
  }
  if (lane == 0) meta[w] = make_int2(cnt, resume);
}

}  // namespace

cudaError_t launch_ot_scan(const void* kT, int lda, int width, const void* t0, const void* t1,
                           const int4* req, int nreq, int K, int32_t* out, int2* meta,
                           cudaStream_t s) {
  if (nreq <= 0) return cudaSuccess;
  const int blocks = (nreq * 32 + 255) / 256;
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    ot_scan_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(kT), lda, static_cast<const T*>(t0), static_cast<const T*>(t1), req, nreq, K, out, meta);
    return 0;
  });
  return cudaGetLastError();
}

}  // namespace otprg
