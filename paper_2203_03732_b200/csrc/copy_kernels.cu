// copy_kernels.cu — copy mode of the assignment solver (
// reference AssignmentOptions::demand_groups / supply_groups,
// assignment.cpp:81-103 scan_grouped and :241-250 the supply-copy lift).
//
// In copy mode the admissible demand vertices of every free b are visited in
// one common order per phase: demand groups ascending; inside a group the
// free copies (ascending id), then the matched copies stable-sorted by their
// partner's supply group.  That order pi is the same for every b, so b-
// proposing deferred acceptance over pi-ordered preferences (lower b wins)
// again reproduces the reference's sequential greedy exactly.  Per phase
// (host-synced; copy mode serves the reference's OT-equivalence checks, not
// the benchmark path):
//   keys + radix sort -> pi and rank      (cub::DeviceRadixSort)
//   DA chains over pi                     (one warp per free b)
//   apply M' (matching, Y(a) -= 1)        exhausted b: Y(b) += 1 in the DA
//   lift free supply copies to their group's maximum dual.
#include <cub/cub.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

// key(a) = (demand group, matched, partner's supply group, a), 21 bits each
__global__ void copy_keys_kernel(const int32_t* __restrict__ dgroup, const int32_t* __restrict__ sgroup,
                                 const int32_t* __restrict__ ma, int n_a,
                                 unsigned long long* __restrict__ keys, int32_t* __restrict__ vals) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_a) return;
  const int b = ma[a];
  const unsigned long long matched = b >= 0 ? 1ull : 0ull;
  const unsigned long long pg = b >= 0 ? (unsigned long long)sgroup[b] : 0ull;
  keys[a] = ((unsigned long long)dgroup[a] << 43) | (matched << 42) | (pg << 21) | (unsigned long long)a;
  vals[a] = a;
}

__global__ void copy_rank_kernel(const int32_t* __restrict__ pi, int n_a, int32_t* __restrict__ rank) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_a) rank[pi[i]] = i;
}

template <typename T>
__device__ __forceinline__ uint32_t elem_of(const T* p, size_t i) {
  return (uint32_t)p[i];
}

// One warp per free b: deferred acceptance with preferences in pi order.
template <typename T>
__global__ void __launch_bounds__(256) copy_da_kernel(const T* __restrict__ kT, int lda,
                                                      const T* __restrict__ t, int32_t* __restrict__ yb,
                                                      const int32_t* __restrict__ ma,
                                                      unsigned long long* __restrict__ holder,
                                                      const int32_t* __restrict__ pi,
                                                      const int32_t* __restrict__ rank,
                                                      const int32_t* __restrict__ bfree, int nfree,
                                                      int n_a, uint32_t phase, int2* __restrict__ mp,
                                                      int* __restrict__ mp_cnt, Ctl* ctl) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nfree) return;
  int b = bfree[w];
  int pos = 0;
  const uint32_t cur_tag = ~phase;
  while (true) {
    const uint32_t target = (uint32_t)yb[b] - 1u;
    int hit = -1;
    for (int i0 = pos & ~31; i0 < n_a; i0 += 32) {
      const int i = i0 + lane;
      bool ok = false;
      if (i >= pos && i < n_a) {
        const int a = pi[i];
        ok = elem_of(kT, (size_t)b * lda + a) + elem_of(t, (size_t)a) == target;
      }
      const unsigned bal = __ballot_sync(kFull, ok);
      if (bal) {
        hit = i0 + __ffs(bal) - 1;
        break;
      }
    }
    if (hit < 0) {  // b stays free: Y(b) += 1 (apply_phase :233-235)
      if (lane == 0) {
        const uint32_t y = (uint32_t)yb[b];
        if (y + 1 > ctl->tmax) report(ctl, 11, (int)phase, b, (int)y);
        yb[b] = (int32_t)(y + 1);
      }
      return;
    }
    const int a = pi[hit];
    const unsigned long long key = ((unsigned long long)cur_tag << 32) | (uint32_t)b;
    unsigned long long old = 0;
    if (lane == 0) old = atomicMin(holder + a, key);
    old = __shfl_sync(kFull, old, 0);
    if (old < key) {  // held by a lower b of this phase
      pos = hit + 1;
      continue;
    }
    if ((uint32_t)(old >> 32) == cur_tag) {  // displaced b2 continues after a
      b = (int)(uint32_t)old;
      pos = rank[a] + 1;
      continue;
    }
    if (lane == 0) {  // first take of a this phase: (a, previous partner)
      const int q = atomicAdd(mp_cnt, 1);
      mp[q] = make_int2(a, ma[a]);
    }
    return;
  }
}

template <typename T>
__global__ void copy_apply_kernel(const int2* __restrict__ mp, const int* __restrict__ mp_cnt,
                                  const unsigned long long* __restrict__ holder, int32_t* __restrict__ ma,
                                  int32_t* __restrict__ mb, T* __restrict__ t, uint32_t phase, Ctl* ctl) {
  const int m = *mp_cnt;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int a = mp[i].x, old_b = mp[i].y;
    const int b = (int)(uint32_t)holder[a];
    if (old_b >= 0) mb[old_b] = -1;
    ma[a] = b;
    mb[b] = a;
    const uint32_t nt = (uint32_t)t[a] + 1u;
    if (nt > ctl->tmax) report(ctl, 12, (int)phase, a, (int)nt);
    t[a] = (T)nt;
  }
}

__global__ void copy_lift_max_kernel(const int32_t* __restrict__ yb, const int32_t* __restrict__ sgroup,
                                     int n_b, int* __restrict__ gmax) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n_b) atomicMax(gmax + sgroup[b], yb[b]);
}

__global__ void copy_lift_set_kernel(int32_t* __restrict__ yb, const int32_t* __restrict__ mb,
                                     const int32_t* __restrict__ sgroup, int n_b,
                                     const int* __restrict__ gmax) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n_b && mb[b] == -1) yb[b] = gmax[sgroup[b]];
}

}  // namespace

size_t copy_sort_temp_bytes(int n_a) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, n_a);
  return bytes;
}

cudaError_t copy_order(const int32_t* dgroup, const int32_t* sgroup, const int32_t* ma, int n_a,
                       unsigned long long* keys, unsigned long long* keys_sorted, int32_t* vals,
                       int32_t* pi, int32_t* rank, void* temp, size_t temp_bytes, cudaStream_t s) {
  const int blocks = (n_a + 255) / 256;
  copy_keys_kernel<<<blocks, 256, 0, s>>>(dgroup, sgroup, ma, n_a, keys, vals);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_sorted, vals, pi, n_a,
                                                  0, 64, s);
  if (e != cudaSuccess) return e;
  copy_rank_kernel<<<blocks, 256, 0, s>>>(pi, n_a, rank);
  return cudaGetLastError();
}

cudaError_t copy_da(const void* kT, int lda, int width, const void* t, int32_t* yb, const int32_t* ma,
                    unsigned long long* holder, const int32_t* pi, const int32_t* rank,
                    const int32_t* bfree, int nfree, int n_a, uint32_t phase, int2* mp, int* mp_cnt,
                    Ctl* ctl, cudaStream_t s) {
  if (nfree <= 0) return cudaSuccess;
  const int blocks = (nfree * 32 + 255) / 256;
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    copy_da_kernel<T><<<blocks, 256, 0, s>>>(static_cast<const T*>(kT), lda, static_cast<const T*>(t), yb,
                                             ma, holder, pi, rank, bfree, nfree, n_a, phase, mp, mp_cnt,
                                             ctl);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t copy_apply(const int2* mp, const int* mp_cnt, const unsigned long long* holder, int32_t* ma,
                       int32_t* mb, void* t, int width, uint32_t phase, Ctl* ctl, cudaStream_t s) {
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    copy_apply_kernel<T><<<148, 256, 0, s>>>(mp, mp_cnt, holder, ma, mb, static_cast<T*>(t), phase, ctl);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t copy_lift(int32_t* yb, const int32_t* mb, const int32_t* sgroup, int n_b, int n_groups,
                      int* gmax, cudaStream_t s) {
  cudaMemsetAsync(gmax, 0x80, sizeof(int) * (size_t)n_groups, s);  // very negative
  const int blocks = (n_b + 255) / 256;
  copy_lift_max_kernel<<<blocks, 256, 0, s>>>(yb, sgroup, n_b, gmax);
  copy_lift_set_kernel<<<blocks, 256, 0, s>>>(yb, mb, sgroup, n_b, gmax);
  return cudaGetLastError();
}

}  // namespace otprg
