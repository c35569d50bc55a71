// solve_kernels.cu — the device-resident phase loop of the push-relabel
// assignment solver (reference: src/assignment.cpp:316-364), for sm_100a.
//
// One persistent cooperative kernel runs whole phases with no host sync.
// Per phase (phase p, free supply set B'_p):
//
//   P step  (reference collect_workset/scan_plain :107-147,65-75 and the
//            sequential greedy :161-171)
//     Every warp repeatedly grabs a free b and runs a deferred-acceptance
//     proposal chain: it scans kT[b][*] (contiguous over a) for the first
//     admissible a >= start (k(a,b) + t(a) == Y(b) - 1, i.e.
//     Y(a)+Y(b) == k+1) and proposes with one 64-bit atomicMin on holder[a]
//     (key = ~phase << 32 | b: lower b wins, stale phases lose).  Rejected ->
//     continue the same row after a.  Winning over a same-phase holder b2 ->
//     the warp takes over b2's chain from a+1.  No admissible a left -> b is
//     unmatched this phase: Y(b) += 1 and b goes to the next free list.
//     Deferred acceptance with a common priority (lower b first) converges to
//     the serial-dictatorship matching regardless of proposal order, which is
//     exactly the reference's sequential greedy M'.
//   A step  (apply_phase :210-235)
//     For every a first held this phase: drop its old partner (which becomes
//     free), link (a, holder b), Y(a) -= 1 (t(a) += 1).
//
// Two grid barriers per phase.  Termination (:330-334) compares the free
// count with floor(eps * min(n_a, n_b)) at the top of the loop; the phase cap
// (:326,356-358) sets status 5.
#include <climits>
#include <cstdio>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

constexpr int kBlock = 1024;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) { return __ldg(p); }

template <bool kSmem>
__device__ __forceinline__ uint4 load_t(const uint4* p) {
  if constexpr (kSmem) return *p;
  else return __ldcg(p);
}

// First admissible a >= start in one kT row, or -1.  The warp streams the
// row in 32 lanes x 16 B x kUnroll chunks (coalesced 128-bit loads, 4 in
// flight per lane).  When track_min, folds min_a (k+t) of every loaded entry
// into mnw (packed per-element minima) for the lazy-skip bound.
template <typename T, bool kSmem>
__device__ __forceinline__ int warp_find_first(const T* __restrict__ row,
                                               const T* tvec, int lda, int start,
                                               uint32_t target, bool track_min,
                                               uint32_t& mnw, int lane,
                                               unsigned long long& bytes) {
  using S = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  constexpr int kBits = 8 * sizeof(T);
  const uint32_t tg = S::rep(target);
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  const uint4* tv = reinterpret_cast<const uint4*>(tvec);
  const int nv = lda / kEpv;  // multiple of 32
  for (int v = (start / kEpv) & ~31; v < nv; v += 32 * kUnroll) {
    uint4 kr[kUnroll], tr[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const int vi = v + j * 32 + lane;
      if (vi < nv) {
        kr[j] = ldg_nc(rv + vi);
        tr[j] = load_t<kSmem>(tv + vi);
      } else {
        kr[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
        tr[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    if (lane == 0) bytes += 16ull * (unsigned long long)min(nv - v, 32 * kUnroll);
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const int vi = v + j * 32 + lane;
      const uint32_t kw[4] = {kr[j].x, kr[j].y, kr[j].z, kr[j].w};
      const uint32_t tw[4] = {tr[j].x, tr[j].y, tr[j].z, tr[j].w};
      int hit = INT_MAX;
#pragma unroll
      for (int w = 3; w >= 0; --w) {  // descending so the lowest word wins
        const uint32_t s = S::add(kw[w], tw[w]);
        uint32_t e = S::eq(s, tg);
        if (track_min) mnw = S::mn(mnw, s);
        const int e0 = vi * kEpv + w * S::kEpw;
        if (e0 < start) {
          const int drop = start - e0;
          e = drop >= S::kEpw ? 0u : (e & (~0u << (drop * kBits)));
        }
        if (e) hit = e0 + (__ffs(e) - 1) / kBits;
      }
      const unsigned bal = __ballot_sync(kFull, hit != INT_MAX);
      if (bal) return __shfl_sync(kFull, hit, __ffs(bal) - 1);
    }
  }
  return -1;
}

// Per-phase pointers (selected once so no parameter array is indexed
// dynamically, which would spill the kernel parameters to local memory).
struct PhasePtrs {
  int32_t* list_nxt;  // free-b list of the next phase
  int32_t* mp_cur;    // a's first held this phase
  int* cnt_nxt;
  int* mp_cnt_cur;
  int* exh_cur;
};

template <typename T, bool kSmem>
__device__ __forceinline__ void run_chain(int b, const SolveArgs& A, const PhasePtrs& P,
                                          const T* tp, int lda, uint32_t phase, uint32_t tmax,
                                          int lane, unsigned long long& bytes,
                                          unsigned long long& steps) {
  using S = Simd<T>;
  Ctl* ctl = A.ctl;
  const T* kT = static_cast<const T*>(A.kT);
  T* rowmin = static_cast<T*>(A.rowmin);
  uint32_t yb = (uint32_t)__ldcg(A.yb + b);
  uint32_t target = yb - 1;
  int start = 0;
  bool fresh = true;
  uint32_t mnw = 0xffffffffu;
  const uint32_t cur_tag = ~phase;
  // Lazy skip: the bound only grows (t only grows), so an empty row stays
  // empty while target < bound.
  bool skip = (uint32_t)__ldcg(rowmin + b) > target;
  while (true) {
    int a = -1;
    if (!skip) {
      a = warp_find_first<T, kSmem>(kT + (size_t)b * lda, tp, lda, start, target, fresh, mnw,
                                    lane, bytes);
      if (lane == 0) ++steps;
#ifdef OTPRG_DEBUG_SCAN
      if (lane == 0) {  // serial re-check of the warp scan
        const T* row = kT + (size_t)b * lda;
        const int hi = a < 0 ? lda : a;
        for (int x = start; x < hi; ++x)
          if ((uint32_t)row[x] + (uint32_t)tp[x] == target)
            report(ctl, 8, (int)phase, b, start, a, x, (int)target);
        if (a >= 0 && (uint32_t)row[a] + (uint32_t)tp[a] != target)
          report(ctl, 9, (int)phase, b, start, a, (int)row[a] * 1000 + (int)tp[a], (int)target);
      }
#endif
    }
    if (a < 0) {
      // b stays free this phase: Y(b) += 1 (apply_phase :233-235).
      uint32_t m = 0;
      if (fresh && !skip) m = __reduce_min_sync(kFull, S::hmin(mnw));
      if (lane == 0) {
        if (fresh && !skip) rowmin[b] = (T)m;
        if (yb + 1 > tmax) report(ctl, 11, (int)phase, b, (int)yb);
        A.yb[b] = (int32_t)(yb + 1);
        const int pos = atomicAdd(P.cnt_nxt, 1);
        P.list_nxt[pos] = b;
        atomicAdd(P.exh_cur, 1);
      }
      return;
    }
    const unsigned long long key = ((unsigned long long)cur_tag << 32) | (uint32_t)b;
    unsigned long long old = 0;
    if (lane == 0) old = atomicMin(A.holder + a, key);
    old = __shfl_sync(kFull, old, 0);
#ifdef OTPRG_DEBUG_SCAN
    if (lane == 0 && (uint32_t)(old >> 32) < cur_tag)  // key from a later phase
      report(ctl, 13, (int)phase, b, a, (int)~(uint32_t)(old >> 32), (int)(uint32_t)old);
#endif
    if (old < key) {  // a is held by a lower b of this phase: next candidate
      start = a + 1;
      continue;
    }
    if ((uint32_t)(old >> 32) == cur_tag) {  // displaced b2 continues after a
      b = (int)(uint32_t)old;
      yb = (uint32_t)__ldcg(A.yb + b);
      target = yb - 1;
      start = a + 1;
      fresh = false;
      skip = false;
      continue;
    }
    if (lane == 0) {  // a newly held this phase
      const int pos = atomicAdd(P.mp_cnt_cur, 1);
      P.mp_cur[pos] = a;
    }
    return;
  }
}

template <typename T, bool kSmem>
__global__ void __launch_bounds__(kBlock, 1) phase_loop_kernel(SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_t = reinterpret_cast<T*>(smem_raw);
  Ctl* ctl = A.ctl;
  const int lda = ctl->lda;
  const int thresh = ctl->thresh;
  const uint32_t cap = (uint32_t)ctl->phase_cap;
  const uint32_t tmax = ctl->tmax;
  uint32_t phase = ld_cg(reinterpret_cast<const unsigned*>(&ctl->phase));
  const int lane = threadIdx.x & 31;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long bytes = 0, steps = 0;
  T* tg = static_cast<T*>(A.t);

  __shared__ int s_ctl[2];
  while (true) {
    const int cur = (phase + 1) & 1, nxt = cur ^ 1;
    // one read per block, broadcast: every thread must take the same branch
    if (threadIdx.x == 0) {
      s_ctl[0] = ld_cg(&ctl->status);
      s_ctl[1] = ld_cg(&ctl->cnt[cur]);
    }
    __syncthreads();
    const int status = s_ctl[0], n = s_ctl[1];
    __syncthreads();
    if (status != 0) break;
    if (n <= thresh) {  // (double)n_i <= eps*m  <=>  n_i <= floor(eps*m)
      if (leader) {
        ctl->done = 1;
        ctl->full_match = (n == 0);
      }
      break;
    }
    if (phase >= A.max_phase) break;
    if (phase + 1 > cap) {
      if (leader) report(ctl, 5, (int)phase);
      break;
    }
    phase += 1;
    // Timeline slots (ns): 0 phase start, 1 t staged, 2/3 last/first block
    // done with P (3 stores ~t), 4 after barrier 1, 5 last block done with A,
    // 6 after barrier 2, 7 n_i.
    unsigned long long* tr =
        (A.trace && phase <= A.trace_cap) ? A.trace + (size_t)(phase - 1) * 8 : nullptr;
    if (leader) {
      A.free_counts[phase - 1] = n;
      ctl->sum_ni += n;
      if (tr) tr[0] = globaltimer(), tr[7] = (unsigned long long)n;
    }
    if constexpr (kSmem) {
      const uint4* src = reinterpret_cast<const uint4*>(tg);
      uint4* dst = reinterpret_cast<uint4*>(s_t);
      const int nvec = lda * (int)sizeof(T) / 16;
      for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = __ldcg(src + i);
      __syncthreads();
    }
    if (tr && leader) tr[1] = globaltimer();
    const T* tp = kSmem ? s_t : tg;

    // ---- P step: proposal chains ----
    const int32_t* list_cur = cur ? A.list[1] : A.list[0];
    PhasePtrs P;
    P.list_nxt = cur ? A.list[0] : A.list[1];
    P.mp_cur = cur ? A.mp[1] : A.mp[0];
    P.cnt_nxt = &ctl->cnt[nxt];
    P.mp_cnt_cur = &ctl->mp_cnt[cur];
    P.exh_cur = &ctl->exh[cur];
    while (true) {
      int i = 0;
      if (lane == 0) i = atomicAdd(&ctl->work[cur], 1);
      i = __shfl_sync(kFull, i, 0);
      if (i >= n) break;
      const int b = __ldcg(list_cur + i);
      run_chain<T, kSmem>(b, A, P, tp, lda, phase, tmax, lane, bytes, steps);
    }
    grid_barrier(ctl, tr ? tr + 2 : nullptr, tr ? tr + 3 : nullptr);
    if (tr && leader) tr[4] = globaltimer();

    // ---- A step: apply M' ----
    const int m = ld_cg(&ctl->mp_cnt[cur]);
    if (leader) {
      // Conservation: every proposer of B' either holds an a (M') or ended
      // unmatched.  A violation means the chains lost or duplicated a b.
      const int x = ld_cg(&ctl->exh[cur]);
      if (x + m != n) report(ctl, 7, (int)phase, n, m, x);
      // Published only after a grid barrier: every block reads ctl->phase
      // once at launch, and a block may start late (cooperative launch only
      // guarantees co-residency, not a common start).
      ctl->phase = phase;
      ctl->work[nxt] = 0;
      ctl->cnt[cur] = 0;
      ctl->mp_cnt[nxt] = 0;
      ctl->exh[nxt] = 0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
      const int a = __ldcg(P.mp_cur + i);
      const unsigned long long key = __ldcg(A.holder + a);
      const int b = (int)(uint32_t)key;
      const int old_b = __ldcg(A.match_a + a);
      if (old_b >= 0) {
        A.match_b[old_b] = -1;
        const int pos = atomicAdd(P.cnt_nxt, 1);
        P.list_nxt[pos] = old_b;
      }
      A.match_a[a] = b;
      A.match_b[b] = a;
      const uint32_t nt = (uint32_t)__ldcg(tg + a) + 1u;
      if (nt > tmax) report(ctl, 12, (int)phase, a, (int)nt);
      tg[a] = (T)nt;
    }
    grid_barrier(ctl, tr ? tr + 5 : nullptr);
    if (tr && leader) tr[6] = globaltimer();
#ifdef OTPRG_DEBUG_SCAN
    if (blockIdx.x == 0) {  // full state consistency after the phase
      __shared__ int s_free, s_bad;
      if (threadIdx.x == 0) s_free = 0, s_bad = -1;
      __syncthreads();
      for (int b = threadIdx.x; b < ctl->n_b; b += blockDim.x) {
        const int a = __ldcg(A.match_b + b);
        if (a == -1) atomicAdd(&s_free, 1);
        else if (__ldcg(A.match_a + a) != b) atomicMax(&s_bad, b);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int nn = ld_cg(&ctl->cnt[nxt]);
        if (s_free != nn || s_bad >= 0) report(ctl, 10, (int)phase, nn, s_free, s_bad);
      }
    }
    grid_barrier(ctl);
#endif
  }
  if (lane == 0 && (bytes | steps)) {
    atomicAdd(&ctl->bytes_touched, bytes);
    atomicAdd(&ctl->chain_steps, steps);
  }
}

template <typename T>
__global__ void init_state_kernel(SolveArgs A, int n_a, int n_b, int lda) {
  T* t = static_cast<T*>(A.t);
  T* rowmin = static_cast<T*>(A.rowmin);
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < lda; i += stride) {
    t[i] = 0;
    if (i < n_a) {
      A.match_a[i] = -1;
      A.holder[i] = ~0ull;
    }
    if (i < n_b) {
      A.match_b[i] = -1;
      A.yb[i] = 1;  // init_state: Y(b) = 1, Y(a) = 0 (assignment.cpp:54-60)
      rowmin[i] = 0;
      A.list[1][i] = i;  // phase 1 proposes every b
    }
  }
}

// Rank-pair completion (complete_matching, assignment.cpp:253-262): the i-th
// free a (ascending) is linked with the i-th free b (ascending).  One block.
__device__ int block_compact_free(const int32_t* match, int n, int32_t* out, int* s_scan) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int chunk = (n + nt - 1) / nt;
  const int lo = min(n, tid * chunk), hi = min(n, lo + chunk);
  int c = 0;
  for (int i = lo; i < hi; ++i) c += (match[i] == -1);
  s_scan[tid] = c;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {  // Hillis-Steele inclusive scan
    const int v = tid >= off ? s_scan[tid - off] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int pos = s_scan[tid] - c;
  const int total = s_scan[nt - 1];
  for (int i = lo; i < hi; ++i)
    if (match[i] == -1) out[pos++] = i;
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(1024) complete_kernel(int32_t* match_a, int32_t* match_b,
                                                        int n_a, int n_b, int32_t* fa,
                                                        int32_t* fb) {
  __shared__ int s_scan[1024];
  const int na_free = block_compact_free(match_a, n_a, fa, s_scan);
  const int nb_free = block_compact_free(match_b, n_b, fb, s_scan);
  const int pairs = min(na_free, nb_free);
  for (int r = threadIdx.x; r < pairs; r += blockDim.x) {
    match_a[fa[r]] = fb[r];
    match_b[fb[r]] = fa[r];
  }
}

__global__ void flush_kernel(uint4* buf, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4((unsigned)i, 0u, 0u, 0u);
}

template <typename T, bool kSmem>
void* loop_fn() {
  return reinterpret_cast<void*>(&phase_loop_kernel<T, kSmem>);
}

void* pick_loop(int width, bool smem_t) {
  if (width == 1) return smem_t ? loop_fn<uint8_t, true>() : loop_fn<uint8_t, false>();
  return smem_t ? loop_fn<uint16_t, true>() : loop_fn<uint16_t, false>();
}

}  // namespace

size_t phase_loop_smem(int width, bool smem_t, int lda) {
  return smem_t ? (size_t)lda * width : 0;
}

bool smem_t_fits(int width, int lda) { return (size_t)lda * width <= 200 * 1024; }

int phase_loop_grid(int width, bool smem_t, int lda, int num_sms) {
  void* fn = pick_loop(width, smem_t);
  const size_t smem = phase_loop_smem(width, smem_t, lda);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem) != cudaSuccess)
    return 0;
  return per_sm * num_sms;
}

cudaError_t launch_phase_loop(const SolveArgs& a, int width, bool smem_t, int lda, int grid,
                              cudaStream_t s) {
  void* fn = pick_loop(width, smem_t);
  SolveArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), params,
                                     phase_loop_smem(width, smem_t, lda), s);
}

cudaError_t launch_init_state(const SolveArgs& a, int n_a, int n_b, int lda, int width,
                              cudaStream_t s) {
  const int blocks = (lda + 255) / 256;
  if (width == 1)
    init_state_kernel<uint8_t><<<blocks, 256, 0, s>>>(a, n_a, n_b, lda);
  else
    init_state_kernel<uint16_t><<<blocks, 256, 0, s>>>(a, n_a, n_b, lda);
  return cudaGetLastError();
}

cudaError_t launch_complete(int32_t* match_a, int32_t* match_b, int n_a, int n_b,
                            int32_t* scratch_a, int32_t* scratch_b, cudaStream_t s) {
  complete_kernel<<<1, 1024, 0, s>>>(match_a, match_b, n_a, n_b, scratch_a, scratch_b);
  return cudaGetLastError();
}

cudaError_t launch_flush(void* buf, size_t bytes, cudaStream_t s) {
  flush_kernel<<<1184, 512, 0, s>>>(static_cast<uint4*>(buf), bytes / 16);
  return cudaGetLastError();
}

}  // namespace otprg
