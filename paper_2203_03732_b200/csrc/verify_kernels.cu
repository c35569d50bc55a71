// verify_kernels.cu — device invariant suite.
//
// verify_feasibility (assignment.cpp:264-312) on the device, in the
// reference's order of checks so the FIRST violation is the one the
// reference would report (report.violations.front(), used by
// check_invariants :344-349):
//   section 0  Matching::validate (core.cpp:69-86): a ascending, then b
//   section 1  per demand a: dual positive, free with nonzero dual, |Y| > bound
//   section 2  per supply b: dual negative, |Y| > bound
//   section 3  every edge, a-major: matched edge not tight (Y(a)+Y(b) != k),
//              otherwise Y(a)+Y(b) > k + 1
// A violation is a 64-bit key (section << 60 | index << 4 | kind); the
// minimum key over the grid (atomicMin) is the reference's first message and
// a counter gives the number of violations.  Two front ends:
//   * the solver's own state (B-major kT of width T, t = -Y(a), int32 Y(b)),
//     between phases of the stepping API — one HBM pass over kT;
//   * arbitrary host state (int32 k row-major, int64 duals) for the
//     free-standing otprg_verify_host (the reference's verify_feasibility
//     signature).
// Plus the admissible-edge lists of every free b (collect_workset's E',
// assignment.cpp:107-147, K = infinity) for the phase observer.
#include <climits>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

__device__ __forceinline__ unsigned long long vkey(unsigned section, unsigned long long index,
                                                   unsigned kind) {
  return ((unsigned long long)section << 60) | (index << 4) | kind;
}

__device__ __forceinline__ void vnote(VerifyOut* o, unsigned long long key, unsigned long long n = 1) {
  atomicMin(&o->first, key);
  atomicAdd(&o->count, n);
}

// Matching::validate: a ascending, then b (indices n_a + b).
__global__ void verify_match_kernel(const int32_t* __restrict__ ma, const int32_t* __restrict__ mb,
                                    int n_a, int n_b, VerifyOut* o) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_a + n_b; i += stride) {
    if (i < n_a) {
      const int b = ma[i];
      if (b == -1) continue;
      if (b < 0 || b >= n_b || mb[b] != i) vnote(o, vkey(0, i, kMatchA));
    } else {
      const int b = i - n_a, a = mb[b];
      if (a == -1) continue;
      if (a < 0 || a >= n_a || ma[a] != b) vnote(o, vkey(0, i, kMatchB));
    }
  }
}

// Dual checks on the solver's state: Y(a) = -t(a) (never positive by
// construction), Y(b) = yb.
template <typename T>
__global__ void verify_duals_kernel(const T* __restrict__ t, const int32_t* __restrict__ yb,
                                    const int32_t* __restrict__ ma, int n_a, int n_b, long long bound,
                                    VerifyOut* o) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_a + n_b; i += stride) {
    if (i < n_a) {
      const long long ya = -(long long)t[i];
      if (ma[i] == -1 && ya != 0) vnote(o, vkey(1, i, kFreeNonzero));
      if ((ya < 0 ? -ya : ya) > bound) vnote(o, vkey(1, i, kDemandBound));
    } else {
      const int b = i - n_a;
      const long long y = yb[b];
      if (y < 0) vnote(o, vkey(2, b, kSupplyNegative));
      if ((y < 0 ? -y : y) > bound) vnote(o, vkey(2, b, kSupplyBound));
    }
  }
}

// Edge checks on the solver's state, one warp per row b of kT.
template <typename T>
__global__ void __launch_bounds__(256) verify_edges_kernel(const T* __restrict__ kT, int lda,
                                                           const T* __restrict__ t,
                                                           const int32_t* __restrict__ yb,
                                                           const int32_t* __restrict__ mb, int n_a,
                                                           int n_b, VerifyOut* o) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b = w; b < n_b; b += nwarps) {
    const long long y = yb[b];
    const int a0 = mb[b];
    // unmatched edge (a,b) violates iff -t(a) + Y(b) > k + 1  <=>  k + t <= Y(b) - 2
    unsigned long long cnt = 0;
    int first = INT_MAX;
    if (y >= 2) {
      const long long thr_ll = y - 2;
      const uint32_t thr = (uint32_t)min(thr_ll, (long long)type_max<T>());
      const uint32_t rep = SD::rep(thr);
      const uint4* rv = reinterpret_cast<const uint4*>(kT + (size_t)b * lda);
      const uint4* tv = reinterpret_cast<const uint4*>(t);
      const int nv = lda / kEpv;
      for (int v0 = 0; v0 < nv; v0 += 32) {
        const int v = v0 + lane;
        uint32_t m = 0;
        if (v < nv) {
          const uint4 k = rv[v], tt = tv[v];
          m = SD::bits(SD::le(SD::add(k.x, tt.x), rep)) |
              (SD::bits(SD::le(SD::add(k.y, tt.y), rep)) << SD::kEpw) |
              (SD::bits(SD::le(SD::add(k.z, tt.z), rep)) << (2 * SD::kEpw)) |
              (SD::bits(SD::le(SD::add(k.w, tt.w), rep)) << (3 * SD::kEpw));
          const int e0 = v * kEpv;
          if (e0 + kEpv > n_a) m &= (n_a > e0) ? ((1u << (n_a - e0)) - 1u) : 0u;  // padding
          if (a0 >= e0 && a0 < e0 + kEpv) m &= ~(1u << (a0 - e0));  // matched edge: below
          if (m) first = min(first, e0 + __ffs(m) - 1);
        }
        cnt += __popc(m);
      }
    }
    if (a0 >= 0 && a0 < n_a) {  // matched edge must be tight: -t(a0) + Y(b) == k
      if (lane == 0 && -(long long)t[a0] + y != (long long)kT[(size_t)b * lda + a0]) {
        vnote(o, vkey(3, (unsigned long long)a0 * n_b + b, kNotTight));
      }
    }
    first = __reduce_min_sync(kFull, first);
    cnt = __reduce_add_sync(kFull, (unsigned)cnt);
    if (lane == 0 && cnt) vnote(o, vkey(3, (unsigned long long)first * n_b + b, kExceeds), cnt);
  }
}

// Host-state variant (int32 k row-major n_a x n_b, int64 duals).
__global__ void verify_host_duals_kernel(const long long* __restrict__ ya,
                                         const long long* __restrict__ yb,
                                         const int32_t* __restrict__ ma, int n_a, int n_b,
                                         long long bound, VerifyOut* o) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_a + n_b; i += stride) {
    if (i < n_a) {
      const long long y = ya[i];
      if (y > 0) vnote(o, vkey(1, i, kDemandPositive));
      if (ma[i] == -1 && y != 0) vnote(o, vkey(1, i, kFreeNonzero));
      if ((y < 0 ? -y : y) > bound) vnote(o, vkey(1, i, kDemandBound));
    } else {
      const int b = i - n_a;
      const long long y = yb[b];
      if (y < 0) vnote(o, vkey(2, b, kSupplyNegative));
      if ((y < 0 ? -y : y) > bound) vnote(o, vkey(2, b, kSupplyBound));
    }
  }
}

__global__ void verify_host_edges_kernel(const int32_t* __restrict__ k, const long long* __restrict__ ya,
                                         const long long* __restrict__ yb,
                                         const int32_t* __restrict__ ma, int n_a, int n_b,
                                         VerifyOut* o) {
  const size_t total = (size_t)n_a * n_b;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int a = (int)(i / n_b), b = (int)(i % n_b);
    const long long sum = ya[a] + yb[b], kv = k[i];
    if (ma[a] == b) {
      if (sum != kv) vnote(o, vkey(3, i, kNotTight));
    } else if (sum > kv + 1) {
      vnote(o, vkey(3, i, kExceeds));
    }
  }
}

// Free supply vertices in ascending order (one block) and their count.
__global__ void __launch_bounds__(1024) free_list_kernel(const int32_t* __restrict__ mb, int n_b,
                                                         int32_t* out, int* count) {
  __shared__ int s_scan[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int chunk = (n_b + nt - 1) / nt;
  const int lo = min(n_b, tid * chunk), hi = min(n_b, lo + chunk);
  int c = 0;
  for (int q = lo; q < hi; ++q) c += (mb[q] == -1);
  s_scan[tid] = c;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {
    const int v = tid >= off ? s_scan[tid - off] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int pos = s_scan[tid] - c;
  for (int q = lo; q < hi; ++q)
    if (mb[q] == -1) out[pos++] = q;
  if (tid == nt - 1) *count = s_scan[nt - 1];
}

// Admissible edges of free b (k + t == Y(b) - 1, a ascending): counts
// (offs == nullptr) or the lists at offs[i] (one warp per free b).
template <typename T>
__global__ void __launch_bounds__(256) admissible_kernel(const T* __restrict__ kT, int lda,
                                                         const T* __restrict__ t,
                                                         const int32_t* __restrict__ yb,
                                                         const int32_t* __restrict__ bfree,
                                                         int nfree, int n_a,
                                                         long long* __restrict__ counts,
                                                         const long long* __restrict__ offs,
                                                         int32_t* __restrict__ out) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nfree) return;
  const int b = bfree[w];
  const long long y = yb[b];
  long long total = 0;
  if (y >= 1 && y - 1 <= (long long)type_max<T>() - 1) {
    const uint32_t rep = SD::rep((uint32_t)(y - 1));
    const uint4* rv = reinterpret_cast<const uint4*>(kT + (size_t)b * lda);
    const uint4* tv = reinterpret_cast<const uint4*>(t);
    const int nv = lda / kEpv;
    for (int v0 = 0; v0 < nv; v0 += 32) {
      const int v = v0 + lane;
      uint32_t m = 0;
      if (v < nv) {
        const uint4 k = rv[v], tt = tv[v];
        m = SD::bits(SD::eq(SD::add(k.x, tt.x), rep)) |
            (SD::bits(SD::eq(SD::add(k.y, tt.y), rep)) << SD::kEpw) |
            (SD::bits(SD::eq(SD::add(k.z, tt.z), rep)) << (2 * SD::kEpw)) |
            (SD::bits(SD::eq(SD::add(k.w, tt.w), rep)) << (3 * SD::kEpw));
        const int e0 = v * kEpv;
        if (e0 + kEpv > n_a) m &= (n_a > e0) ? ((1u << (n_a - e0)) - 1u) : 0u;
      }
      const int c = __popc(m);
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += yv;
      }
      if (offs && m) {
        long long idx = offs[w] + total + inc - c;
        const int e0 = v * kEpv;
        while (m) {
          out[idx++] = e0 + __ffs(m) - 1;
          m &= m - 1;
        }
      }
      total += __shfl_sync(kFull, inc, 31);
    }
  }
  if (!offs && lane == 0) counts[w] = total;
}

}  // namespace

cudaError_t launch_verify_state(const void* kT, int lda, int width, const void* t,
                                const int32_t* yb, const int32_t* ma, const int32_t* mb, int n_a,
                                int n_b, long long bound, VerifyOut* out, cudaStream_t s) {
  const int blocks = 148 * 4;
  verify_match_kernel<<<blocks, 256, 0, s>>>(ma, mb, n_a, n_b, out);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    verify_duals_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(t), yb, ma, n_a, n_b, bound, out);
    verify_edges_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(kT), lda, static_cast<const T*>(t),
                                                  yb, mb, n_a, n_b, out);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_verify_host(const int32_t* k, const long long* ya, const long long* yb,
                               const int32_t* ma, const int32_t* mb, int n_a, int n_b,
                               long long bound, VerifyOut* out, cudaStream_t s) {
  const int blocks = 148 * 4;
  verify_match_kernel<<<blocks, 256, 0, s>>>(ma, mb, n_a, n_b, out);
  verify_host_duals_kernel<<<blocks, 256, 0, s>>>(ya, yb, ma, n_a, n_b, bound, out);
  verify_host_edges_kernel<<<blocks, 256, 0, s>>>(k, ya, yb, ma, n_a, n_b, out);
  return cudaGetLastError();
}

cudaError_t launch_free_list(const int32_t* mb, int n_b, int32_t* out, int* count, cudaStream_t s) {
  free_list_kernel<<<1, 1024, 0, s>>>(mb, n_b, out, count);
  return cudaGetLastError();
}

cudaError_t launch_admissible(const void* kT, int lda, int width, const void* t, const int32_t* yb,
                              const int32_t* bfree, int nfree, int n_a, long long* counts,
                              const long long* offs, int32_t* out, cudaStream_t s) {
  if (nfree <= 0) return cudaSuccess;
  const int blocks = (nfree * 32 + 255) / 256;
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    admissible_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(kT), lda, static_cast<const T*>(t), yb, bfree, nfree, n_a, counts, offs, out);
    return 0;
  });
  return cudaGetLastError();
}

}  // namespace otprg
