// ot_device.cu — the OT copy/cluster phase on the device (SURVEY §8(a) O2/O3,
// kernels K10/K11; reference semantics: solve_copy_matching, src/ot.cpp:418-637).
//
// State (every vertex carries at most two dual clusters, ot.hpp:65-96):
//   demand cluster code = 2a + slot (slot 0 the higher dual; count 0 = absent):
//     dy, dfree, dmatched; its flow (b, copies) ascending b in CSR by code,
//     followed by one sentinel entry b = kFreeB holding the free copies;
//   supply cluster 2b + slot (slot 0 the higher dual): sy, sfree, smatched.
//
// One phase:
//   free list    supply vertices with free copies, ascending b, their dual y_b
//                and copy count; n_i for the termination test;
//   admissible   every free b's admissible clusters, y(a,ci) = k(a,b)+1-y_b,
//                ascending a (CSR; count pass + fill pass over kT rows);
//   claim (K10)  capacitated deferred acceptance: each b proposes its
//                unplaced copies to its frontier cluster; a cluster keeps the
//                lowest b's up to its capacity (free + matched copies at phase
//                start) and returns the rest; a b rejected at its frontier
//                moves on, copies returned from an earlier cluster go to the
//                frontier again.  With one priority order (b ascending) over
//                every cluster this reaches exactly the reference's greedy
//                claims (b ascending, each taking min(remaining, available)
//                from its admissible clusters in ascending a; checked against
//                a serial restatement on random instances and by the goldens);
//   update (K11) a cluster that gave c copies lost min(c, free) free copies
//                and its first c - min(c, free) matched copies in ascending
//                partner order (ot.cpp:504-514); the displaced partners' copies
//                return free at their old dual k(a,b_old) - y; the claiming
//                b's copies join the cluster one dual below; supply copies
//                left free go up a unit; then both sides are normalised
//                (free supply copies lifted to the vertex maximum, equal duals
//                merged, empty clusters dropped, at most two per vertex,
//                ot.cpp:362-414) — by one sort of all flow records keyed
//                (a, descending y, b) and per-vertex passes.
// Errors (the reference's InvariantViolation messages) are reported as status
// 5 with a code in err[0]: 1 third demand dual, 2 third supply dual, 3
// displaced copy without a supply cluster, 4 storage bound exceeded.
#include <climits>
#include <cstdlib>
#include <cub/cub.cuh>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

__device__ __forceinline__ void ot_fail(OtDev& D, int code, int x = 0, int y = 0) {
  if (atomicCAS(D.status, 0, 5) == 0) {
    D.err[0] = code;
    D.err[1] = x;
    D.err[2] = y;
  }
}

// The device-sized phase stopped for the host (kCtrHold): later steps return.
// (inside the persistent loop the loop itself tests the hold between steps,
// so the steps skip this round trip)
__device__ __forceinline__ bool ot_hold(const OtDev& D) {
  return !D.in_loop && *(volatile int64_t*)&D.ctr[kCtrHold] != 0;
}

template <typename T>
__device__ __forceinline__ uint32_t k_at(const OtDev& D, int a, int b) {
  return static_cast<const T*>(D.kT)[(size_t)b * D.lda + a];
}

// ---- free list ---------------------------------------------------------------
// Per supply vertex: total free copies (after normalisation at most one slot
// holds free copies: the vertex maximum).
__device__ __forceinline__ int64_t sfree_total(const OtDev& D, int b) {
  return D.sfree[2 * b] + D.sfree[2 * b + 1];
}

constexpr int kListBlocks = 148;

__device__ __forceinline__ void ot_free_count_body(OtDev& D, int* counts, int bid, int nb) {
  if (ot_hold(D)) return;
  const int n = D.n_b, chunk = (n + nb - 1) / nb;
  const int lo = min(n, bid * chunk), hi = min(n, lo + chunk);
  int c = 0;
  long long tot = 0;
  for (int b = lo + threadIdx.x; b < hi; b += blockDim.x) {
    const int64_t f = sfree_total(D, b);
    c += f > 0;
    tot += f;
  }
  __shared__ int s_c;
  __shared__ unsigned long long s_t;
  if (threadIdx.x == 0) s_c = 0, s_t = 0;
  __syncthreads();
  c = __reduce_add_sync(kFull, c);
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
  if ((threadIdx.x & 31) == 0) {
    if (c) atomicAdd(&s_c, c);
    if (tot) atomicAdd(&s_t, (unsigned long long)tot);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    counts[bid] = s_c;
    if (s_t) atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrNi]), s_t);
  }
}
__global__ void __launch_bounds__(1024) ot_free_count_kernel(OtDev D, int* counts) {
  ot_free_count_body(D, counts, blockIdx.x, gridDim.x);
}

__device__ __forceinline__ void ot_free_write_body(OtDev& D, const int* counts, int bid, int nb) {
  if (ot_hold(D)) return;
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int n = D.n_b, chunk = (n + nb - 1) / nb;
  const int lo = min(n, bid * chunk), hi = min(n, lo + chunk);
  if (threadIdx.x == 0) {
    int off = 0;
    for (int g = 0; g < bid; ++g) off += counts[g];
    s_base = off;
    if (bid == nb - 1) D.ctr[kCtrFree] = off + counts[bid];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int t0 = lo; t0 < hi; t0 += blockDim.x) {
    const int b = t0 + threadIdx.x;
    int64_t f = 0;
    if (b < hi) f = sfree_total(D, b);
    const bool on = f > 0;
    const unsigned bal = __ballot_sync(kFull, on);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nwarps; ++w) {
      if (w < warp) before += s_warp[w];
      total += s_warp[w];
    }
    if (b < hi) D.fidx[b] = -1;
    if (on) {
      const int pos = s_base + before + __popc(bal & ((1u << lane) - 1u));
      D.fb[pos] = b;
      D.fu0[pos] = f;
      D.fu[pos] = f;
      D.fpos[pos] = 0;
      D.fy[pos] = D.sfree[2 * b] > 0 ? D.sy[2 * b] : D.sy[2 * b + 1];
      D.fidx[b] = pos;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(1024) ot_free_write_kernel(OtDev D, const int* counts) {
  ot_free_write_body(D, counts, blockIdx.x, gridDim.x);
}

// t_ci(a) = -y of cluster (a, ci), type max when absent (never admissible).
template <typename T>
__device__ __forceinline__ void ot_t_body(OtDev& D, int bid, int nb) {
  T* t = static_cast<T*>(D.t);
  for (int a = bid * blockDim.x + threadIdx.x; a < D.lda; a += nb * blockDim.x)
    for (int s = 0; s < 2; ++s) {
      uint32_t v = type_max<T>();
      if (a < D.n_a && D.dfree[2 * a + s] + D.dmatched[2 * a + s] > 0) {
        const int64_t ty = -(int64_t)D.dy[2 * a + s];
        if (ty < 0 || ty > (int64_t)type_max<T>() - 2) ot_fail(D, 4, a, (int)ty);
        else v = (uint32_t)ty;
      }
      t[(size_t)s * D.lda + a] = (T)v;
    }
}
template <typename T>
__global__ void ot_t_kernel(OtDev D) { ot_t_body<T>(D, blockIdx.x, gridDim.x); }

// ---- admissible clusters (warp per free b, full row) ---------------------------
// pass 0: count; pass 1: write codes 2a + ci ascending a at adm_off[i].
template <typename T, int kPass>
__device__ __forceinline__ void ot_adm_body(OtDev& D, int bid, int nb) {
  using S = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  if (ot_hold(D)) return;
  const int nf = D.ctr[kCtrFree];
  if (kPass && D.adm_cap > 0 && D.adm_off[nf] > D.adm_cap) {  // (device-sized phase) the host grows adm
    if (bid == 0 && threadIdx.x == 0) D.ctr[kCtrHold] = 1;
    return;
  }
  const int nwarps = (nb * blockDim.x) >> 5;
  const uint4* v0 = static_cast<const uint4*>(D.t);
  const uint4* v1 = reinterpret_cast<const uint4*>(static_cast<const T*>(D.t) + D.lda);
  const int nv = D.lda / kEpv;
  for (int i = (bid * blockDim.x + threadIdx.x) >> 5; i < nf; i += nwarps) {
    const int b = D.fb[i];
    const uint32_t tg = S::rep((uint32_t)(D.fy[i] - 1));
    const uint4* rv = reinterpret_cast<const uint4*>(static_cast<const T*>(D.kT) + (size_t)b * D.lda);
    int64_t pos = kPass ? D.adm_off[i] : 0;
    int cnt = 0;
    for (int v0i = 0; v0i < nv; v0i += 32) {
      const int vi = v0i + lane;
      uint32_t m0 = 0, m1 = 0;
      if (vi < nv) {
        const uint4 k = __ldg(rv + vi), x0 = __ldg(v0 + vi), x1 = __ldg(v1 + vi);
        const uint32_t kw[4] = {k.x, k.y, k.z, k.w}, w0[4] = {x0.x, x0.y, x0.z, x0.w},
                       w1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          m0 |= S::bits(S::eq(S::add(kw[q], w0[q]), tg)) << (q * S::kEpw);
          m1 |= S::bits(S::eq(S::add(kw[q], w1[q]), tg)) << (q * S::kEpw);
        }
      }
      const uint32_t m = m0 | m1;  // (the two clusters of a have distinct duals: one bit per a at most)
      const int c = __popc(m);
      if (!__ballot_sync(kFull, c != 0)) continue;
      int inc = c;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(kFull, inc, s);
        if (lane >= s) inc += y;
      }
      if (kPass) {
        int64_t o = pos + inc - c;
        uint32_t bm = m;
        while (bm) {
          const int e = __ffs(bm) - 1;
          bm &= bm - 1;
          const int a = vi * kEpv + e;
          D.adm[o++] = 2 * a + ((m1 >> e) & 1);
        }
      }
      const int tot = __shfl_sync(kFull, inc, 31);
      cnt += tot;
      pos += tot;
    }
    if (!kPass && lane == 0) D.adm_len[i] = cnt;
  }
}
template <typename T, int kPass>
__global__ void __launch_bounds__(256) ot_adm_kernel(OtDev D) { ot_adm_body<T, kPass>(D, blockIdx.x, gridDim.x); }

// ---- deferred acceptance -------------------------------------------------------
// Entries: key = (code << 21) | list index, value = copies.
// cl_cut[c]: when cluster c is full, the highest list index among its holders
// (-1: capacity 0); INT_MAX while it has room.  A b above the cut would be
// rejected there, so it skips the cluster without a round (the cut only falls
// once set, so a stale value only skips less).
__device__ __forceinline__ void ot_cut_init_body(OtDev& D, int bid, int nb) {
  if (ot_hold(D)) return;
  for (int c = bid * blockDim.x + threadIdx.x; c < 2 * D.n_a; c += nb * blockDim.x)
    D.cl_cut[c] = D.dfree[c] + D.dmatched[c] > 0 ? INT_MAX : -1;
}
__global__ void ot_cut_init_kernel(OtDev D) { ot_cut_init_body(D, blockIdx.x, gridDim.x); }

__global__ void ot_da_propose_kernel(OtDev D) {
  const int nf = D.ctr[kCtrFree];
  const long long base = D.ctr[kCtrE];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    const int64_t u = D.fu[i];
    if (u <= 0) continue;
    int p = D.fpos[i];
    const int len = (int)D.adm_len[i];
    const int32_t* list = D.adm + D.adm_off[i];
    while (p < len && __ldcg(&D.cl_cut[list[p]]) < i) ++p;  // full of lower b's: rejected anyway
    D.fpos[i] = p;
    if (p >= len) continue;  // admissible set exhausted: these copies stay free
    const int code = list[p];
    const long long slot = base + atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrNew]), 1ull);
    D.e_key[slot] = ((unsigned long long)(uint32_t)code << 21) | (uint32_t)i;
    D.e_val[slot] = u;
    D.fu[i] = 0;
  }
}

// After the sort: every run of equal keys (a b that re-proposed to a cluster it
// holds) is summed into its last entry; within a cluster's segment the copies
// of lower b's come first.  The entry keeps min(amount, capacity left); the
// rest returns to its b, which leaves a frontier cluster that rejected it.
__global__ void ot_da_resolve_kernel(OtDev D, const unsigned long long* __restrict__ key,
                                     const int64_t* __restrict__ val, long long n,
                                     unsigned long long* __restrict__ out_key, int64_t* __restrict__ out_val) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const unsigned long long kj = key[j];
    if (j + 1 < n && key[j + 1] == kj) continue;  // the run's last entry carries it
    const uint32_t code = (uint32_t)(kj >> 21);
    const int i = (int)(kj & ((1u << 21) - 1));
    int64_t amt = val[j], pre = 0;
    long long q = j - 1;
    for (; q >= 0 && key[q] == kj; --q) amt += val[q];
    for (; q >= 0 && (uint32_t)(key[q] >> 21) == code; --q) pre += val[q];
    const int64_t cap = D.dfree[code] + D.dmatched[code];
    const int64_t acc = max((int64_t)0, min(amt, cap - pre));
    const int64_t rej = amt - acc;
    if (acc > 0 && pre + acc == cap) D.cl_cut[code] = i;  // full: holders up to list index i
    if (rej > 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&D.fu[i]), (unsigned long long)rej);
      const int p = D.fpos[i];
      if (p < D.adm_len[i] && D.adm[D.adm_off[i] + p] == (int)code) D.fpos[i] = p + 1;
    }
    if (acc > 0) {
      const long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrE]), 1ull);
      out_key[slot] = kj;
      out_val[slot] = acc;
    }
  }
}

// ---- device-sized rounds ---------------------------------------------------------
// The same round without a sort or a host size: the entries (survivors in
// e_key[0, E), this round's proposals after them) are grouped by cluster into
// per-cluster segments of s_key (count, allocate, scatter), then one warp per
// cluster proposed to ranks its entries by list index and resolves them
// exactly as ot_da_resolve_kernel does on the sorted run.  Every kernel
// returns at once when the rounds are over (ctr[kCtrDone]), so a batch of
// rounds is launched without looking at the counters.
__device__ __forceinline__ bool da_over(const OtDev& D) {
  return !D.in_loop && (*(volatile int64_t*)&D.ctr[kCtrDone] != 0 || ot_hold(D));
}

__device__ __forceinline__ void ot_da_propose_batched_body(OtDev& D, int bid, int nb) {
  if (da_over(D)) return;
  if (bid == 0 && threadIdx.x == 0) {  // (unused by propose; reset for this round's count / alloc)
    D.ctr[kCtrTouch] = 0;
    D.ctr[kCtrAlloc] = 0;
  }
  const int nf = D.ctr[kCtrFree];
  const long long base = D.ctr[kCtrE];
  for (int i = bid * blockDim.x + threadIdx.x; i < nf; i += nb * blockDim.x) {
    const int64_t u = D.fu[i];
    if (u <= 0) continue;
    int p = D.fpos[i];
    const int len = (int)D.adm_len[i];
    const int32_t* list = D.adm + D.adm_off[i];
    while (p < len && __ldcg(&D.cl_cut[list[p]]) < i) ++p;
    D.fpos[i] = p;
    if (p >= len) continue;
    const int code = list[p];
    const long long slot = base + atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrNew]), 1ull);
    D.e_key[slot] = ((unsigned long long)(uint32_t)code << 21) | (uint32_t)i;
    D.e_val[slot] = u;
    D.fu[i] = 0;
  }
}
__global__ void ot_da_propose_batched_kernel(OtDev D) { ot_da_propose_batched_body(D, blockIdx.x, gridDim.x); }

__device__ __forceinline__ void ot_da_count_body(OtDev& D, int bid, int nb) {
  if (da_over(D)) return;
  const long long nn = D.ctr[kCtrNew];
  if (nn == 0) {  // no b has copies to place and a cluster to try: the claims are final
    if (bid == 0 && threadIdx.x == 0) D.ctr[kCtrDone] = 1;
    return;
  }
  if (bid == 0 && threadIdx.x == 0) ++D.ctr[kCtrRounds];
  const long long n = D.ctr[kCtrE] + nn;
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x) {
    const int code = (int)(D.e_key[j] >> 21);
    if (atomicAdd(&D.da_cnt[code], 1) == 0)
      D.da_touch[atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrTouch]), 1ull)] = code;
  }
}
__global__ void ot_da_count_kernel(OtDev D) { ot_da_count_body(D, blockIdx.x, gridDim.x); }

__device__ __forceinline__ void ot_da_alloc_body(OtDev& D, int bid, int nb) {
  if (da_over(D)) return;
  if (bid == 0 && threadIdx.x == 0) {  // (nobody below reads E / New)
    D.ctr[kCtrN] = D.ctr[kCtrE] + D.ctr[kCtrNew];
    D.ctr[kCtrE] = 0;
  }
  const int nt = (int)D.ctr[kCtrTouch];
  const int lane = threadIdx.x & 31;
  // whole warps iterate (one aggregated atomic per warp)
  for (int t0 = (bid * blockDim.x + threadIdx.x) & ~31; t0 < nt; t0 += nb * blockDim.x) {
    const int t = t0 + lane;
    int code = -1, c = 0;
    if (t < nt) {
      code = D.da_touch[t];
      c = D.da_cnt[code];
      if (c > kDaWarpMax) D.ctr[kCtrBig] = 1;  // this round goes the sorted way
    }
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrAlloc]), (unsigned long long)inc);
    base = __shfl_sync(kFull, base, 31);
    if (code >= 0) D.da_off[code] = (int64_t)(base + inc - c);
  }
}
__global__ void ot_da_alloc_kernel(OtDev D) { ot_da_alloc_body(D, blockIdx.x, gridDim.x); }

__device__ __forceinline__ void ot_da_scatter_body(OtDev& D, int bid, int nb) {
  if (da_over(D)) return;
  if (D.ctr[kCtrBig]) {  // (set by the allocation: every block sees it)
    if (bid == 0 && threadIdx.x == 0) D.ctr[kCtrDone] = 2;
    return;
  }
  const long long n = D.ctr[kCtrN];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x) {
    const unsigned long long k = D.e_key[j];
    const int code = (int)(k >> 21);
    const long long pos = D.da_off[code] + atomicAdd(&D.da_fill[code], 1);
    D.s_key[pos] = k;
    D.s_val[pos] = D.e_val[j];
  }
}
__global__ void ot_da_scatter_kernel(OtDev D) { ot_da_scatter_body(D, blockIdx.x, gridDim.x); }

__device__ __forceinline__ void ot_da_resolve_warp_body(OtDev& D, int bid, int nb) {
  if (da_over(D)) return;
  if (bid == 0 && threadIdx.x == 0) D.ctr[kCtrNew] = 0;  // (count has read it) next round's proposals
  const int lane = threadIdx.x & 31;
  const int nt = (int)D.ctr[kCtrTouch];
  const int warps = nb * (blockDim.x >> 5);
  for (int t = bid * (blockDim.x >> 5) + (threadIdx.x >> 5); t < nt; t += warps) {
    const int code = D.da_touch[t];
    const int c = D.da_cnt[code];
    const long long o = D.da_off[code];
    const int64_t cap = D.dfree[code] + D.dmatched[code];
    for (int b0 = 0; b0 < c; b0 += 32) {
      const int e = b0 + lane;
      const bool valid = e < c;
      const unsigned long long ke = valid ? D.s_key[o + e] : 0ull;
      const int ie = valid ? (int)(ke & ((1u << 21) - 1)) : INT_MAX;
      int64_t amt = 0, pre = 0;
      bool last = true;
      for (int b1 = 0; b1 < c; b1 += 32) {
        const int e2 = b1 + lane;
        const int i2 = e2 < c ? (int)(D.s_key[o + e2] & ((1u << 21) - 1)) : INT_MAX;
        const int64_t v2 = e2 < c ? D.s_val[o + e2] : 0;
        const int m = min(32, c - b1);
        for (int q = 0; q < m; ++q) {
          const int iq = __shfl_sync(0xffffffffu, i2, q);
          const int64_t vq = __shfl_sync(0xffffffffu, v2, q);
          if (iq < ie) pre += vq;
          else if (iq == ie) {
            amt += vq;
            if (b1 + q > e) last = false;  // a later duplicate carries the run
          }
        }
      }
      if (!valid || !last) continue;
      const int i = ie;
      const int64_t acc = max((int64_t)0, min(amt, cap - pre));
      const int64_t rej = amt - acc;
      if (acc > 0 && pre + acc == cap) D.cl_cut[code] = i;
      if (rej > 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&D.fu[i]), (unsigned long long)rej);
        const int p = D.fpos[i];
        if (p < D.adm_len[i] && D.adm[D.adm_off[i] + p] == code) D.fpos[i] = p + 1;
      }
      if (acc > 0) {
        const long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrE]), 1ull);
        D.e_key[slot] = ke;
        D.e_val[slot] = acc;
      }
    }
    __syncwarp();
    if (lane == 0) {
      D.da_cnt[code] = 0;
      D.da_fill[code] = 0;
    }
  }
}
__global__ void ot_da_resolve_warp_kernel(OtDev D) { ot_da_resolve_warp_body(D, blockIdx.x, gridDim.x); }

// After a round that went the sorted way: the per-cluster counts back to 0.
__global__ void ot_da_clear_kernel(OtDev D) {
  const int nt = (int)D.ctr[kCtrTouch];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const int code = D.da_touch[t];
    D.da_cnt[code] = 0;
    D.da_fill[code] = 0;
  }
}

// ---- updates -------------------------------------------------------------------
// Copies each demand cluster gave this phase (final claims sorted by code).
__device__ __forceinline__ void ot_consumed_body(OtDev& D, const unsigned long long* __restrict__ key,
                                   const int64_t* __restrict__ val, long long n, int bid, int nb) {
  if (ot_hold(D)) return;
  if (n < 0) n = D.ctr[kCtrE];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&D.consumed[key[j] >> 21]), (unsigned long long)val[j]);
}
__global__ void ot_consumed_kernel(OtDev D, const unsigned long long* __restrict__ key,
                                   const int64_t* __restrict__ val, long long n) {
  ot_consumed_body(D, key, val, n, blockIdx.x, gridDim.x);
}

// Records of the next state, key (a, descending y, b), b = kFreeB for free
// demand copies: surviving flow entries (the displaced prefix removed, its
// supply copies freed at their old dual), the free copies left, the claims
// one dual below.
constexpr uint32_t kYBias = 1u << 20;
__device__ __forceinline__ unsigned long long rec_key(int a, int y, int b) {
  const unsigned long long bk = b == kFreeB ? (1ull << 21) - 1 : (unsigned long long)b;
  return ((unsigned long long)a << 42) | ((unsigned long long)(kYBias - y) << 21) | bk;
}

__device__ __forceinline__ void put_rec(OtDev& D, int a, int y, int b, int64_t cnt) {
  const long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(&D.ctr[kCtrRec]), 1ull);
  D.r_key[slot] = rec_key(a, y, b);
  D.r_val[slot] = cnt;
}

template <typename T>
__device__ __forceinline__ void ot_flow_records_body(OtDev& D, int bid, int nb) {
  if (ot_hold(D)) return;
  const long long nfl = D.fl_off[2 * D.n_a];
  for (long long f = bid * (long long)blockDim.x + threadIdx.x; f < nfl; f += (long long)nb * blockDim.x) {
    const int code = D.fl_code[f];
    const int a = code >> 1, y = D.dy[code], b = D.fl_b[f];
    const int64_t cnt = D.fl_cnt[f];
    const int64_t cons = D.consumed[code];
    if (b == kFreeB) {  // free copies go first
      const int64_t left = cnt - min(cons, cnt);
      if (left > 0) put_rec(D, a, y, kFreeB, left);
      continue;
    }
    // matched copies, ascending partner: displaced are the first cons - free of them
    const int64_t free_c = D.dfree[code];
    const int64_t disp_total = max((int64_t)0, cons - free_c);
    const int64_t before = D.fl_pre[f];
    const int64_t disp = max((int64_t)0, min(cnt, disp_total - before));
    if (cnt - disp > 0) put_rec(D, a, y, b, cnt - disp);
    if (disp > 0) {  // the partner's copies return free at their old dual k(a,b) - y (ot.cpp:560-575)
      const int y_old = (int)k_at<T>(D, a, b) - y;
      int s = -1;
      for (int q = 0; q < 2; ++q)
        if (D.sfree[2 * b + q] + D.smatched[2 * b + q] > 0 && D.sy[2 * b + q] == y_old) s = q;
      if (s < 0) {
        ot_fail(D, 3, a, b);
        continue;
      }
      atomicAdd(reinterpret_cast<unsigned long long*>(&D.sfreed[2 * b + s]), (unsigned long long)disp);
    }
  }
}
template <typename T>
__global__ void ot_flow_records_kernel(OtDev D) { ot_flow_records_body<T>(D, blockIdx.x, gridDim.x); }

__device__ __forceinline__ void ot_claim_records_body(OtDev& D, const unsigned long long* __restrict__ key,
                                        const int64_t* __restrict__ val, long long n, int bid, int nb) {
  if (ot_hold(D)) return;
  if (n < 0) n = D.ctr[kCtrE];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x) {
    const int code = (int)(key[j] >> 21), i = (int)(key[j] & ((1u << 21) - 1));
    put_rec(D, code >> 1, D.dy[code] - 1, D.fb[i], val[j]);
  }
}
__global__ void ot_claim_records_kernel(OtDev D, const unsigned long long* __restrict__ key,
                                        const int64_t* __restrict__ val, long long n) {
  ot_claim_records_body(D, key, val, n, blockIdx.x, gridDim.x);
}

// Supply side (ot.cpp:540-553, 580-588): a free b's copies placed this phase
// join its free cluster's matched copies, the rest go up a unit; displaced
// copies come back free at their cluster; then normalize_supply: every free
// copy lifted to the vertex maximum dual, equal duals merged, empty dropped,
// at most two clusters (slot 0 the higher dual).
__device__ __forceinline__ void ot_supply_body(OtDev& D, int bid, int nb) {
  if (ot_hold(D)) return;
  for (int b = bid * blockDim.x + threadIdx.x; b < D.n_b; b += nb * blockDim.x) {
    int y[3];
    int64_t fr[3], mt[3];
    int n = 0;
    const int i = D.fidx[b];
    for (int s = 0; s < 2; ++s) {
      int64_t f = D.sfree[2 * b + s], m = D.smatched[2 * b + s];
      const int64_t back = D.sfreed[2 * b + s];
      D.sfreed[2 * b + s] = 0;
      if (f + m == 0) continue;
      if (i >= 0 && f > 0) {  // this phase's free cluster
        m += D.fu0[i] - D.fu[i];
        f = 0;
      }
      m -= back;  // displaced copies leave the matched count ...
      f += back;  // ... and come back free at this dual
      if (m < 0) ot_fail(D, 3, -1, b);
      y[n] = D.sy[2 * b + s];
      fr[n] = f;
      mt[n] = m;
      ++n;
    }
    if (i >= 0 && D.fu[i] > 0) {  // copies left free: one dual up
      y[n] = D.fy[i] + 1;
      fr[n] = D.fu[i];
      mt[n] = 0;
      ++n;
    }
    // normalize_supply
    int64_t free_tot = 0;
    int ymax = INT_MIN;
    for (int q = 0; q < n; ++q)
      if (fr[q] + mt[q] > 0) {
        free_tot += fr[q];
        ymax = max(ymax, y[q]);
      }
    int oy[2] = {0, 0};
    int64_t ofr[2] = {0, 0}, omt[2] = {0, 0};
    int m = 0;
    auto add = [&](int yy, int64_t f, int64_t mm) {
      for (int q = 0; q < m; ++q)
        if (oy[q] == yy) {
          ofr[q] += f;
          omt[q] += mm;
          return;
        }
      if (m == 2) {
        ot_fail(D, 2, b);
        return;
      }
      oy[m] = yy;
      ofr[m] = f;
      omt[m] = mm;
      ++m;
    };
    for (int q = 0; q < n; ++q)
      if (mt[q] > 0) add(y[q], 0, mt[q]);
    if (free_tot > 0) add(ymax, free_tot, 0);
    if (m == 2 && oy[1] > oy[0]) {
      const int ty = oy[0];
      oy[0] = oy[1];
      oy[1] = ty;
      const int64_t tf = ofr[0], tm = omt[0];
      ofr[0] = ofr[1];
      omt[0] = omt[1];
      ofr[1] = tf;
      omt[1] = tm;
    }
    for (int q = 0; q < 2; ++q) {
      D.sy[2 * b + q] = q < m ? oy[q] : INT_MIN;
      D.sfree[2 * b + q] = q < m ? ofr[q] : 0;
      D.smatched[2 * b + q] = q < m ? omt[q] : 0;
    }
  }
}
__global__ void ot_supply_kernel(OtDev D) { ot_supply_body(D, blockIdx.x, gridDim.x); }

// After the records are sorted and merged (unique keys, summed counts): the
// record's demand slot (0 for the vertex's first dual, 1 for the second; a
// third is the reference's "third dual value" violation) and its code.
__device__ __forceinline__ void ot_slot_body(OtDev& D, const unsigned long long* __restrict__ key, long long n,
                                             int bid, int nb) {
  if (ot_hold(D)) return;
  if (n < 0) n = D.ctr[kCtrNFlows];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x) {
    const unsigned long long kj = key[j];
    const unsigned long long a = kj >> 42, yk = (kj >> 21) & ((1ull << 21) - 1);
    // first record of a: lower_bound of (a, 0, 0)
    long long lo = 0, hi = j;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if ((key[mid] >> 42) < a) lo = mid + 1;
      else hi = mid;
    }
    const unsigned long long yk0 = (key[lo] >> 21) & ((1ull << 21) - 1);
    int slot = 0;
    if (yk != yk0) {
      // first record of a with a different dual
      long long l2 = lo, h2 = j;
      while (l2 < h2) {
        const long long mid = (l2 + h2) >> 1;
        if (((key[mid] >> 21) & ((1ull << 21) - 1)) == yk0) l2 = mid + 1;
        else h2 = mid;
      }
      slot = (((key[l2] >> 21) & ((1ull << 21) - 1)) == yk) ? 1 : 2;
      if (slot == 2) ot_fail(D, 1, (int)a);
    }
    D.fl_code[j] = (int)(2 * a) + min(slot, 1);
  }
}
__global__ void ot_slot_kernel(OtDev D, const unsigned long long* __restrict__ key, long long n) {
  ot_slot_body(D, key, n, blockIdx.x, gridDim.x);
}

// New CSR: fl_off[c] = first record of code c (lower bound), cluster fields
// from the code's segment, the flow prefix sums for the next displacement.
__device__ __forceinline__ void ot_rebuild_body(OtDev& D, const unsigned long long* __restrict__ key,
                                  const int64_t* __restrict__ val, long long n, int bid, int nb) {
  if (ot_hold(D)) return;
  if (n < 0) n = D.ctr[kCtrNFlows];
  const int nc = 2 * D.n_a;
  for (int c = bid * blockDim.x + threadIdx.x; c <= nc; c += nb * blockDim.x) {
    long long lo = 0, hi = n;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (D.fl_code[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    D.fl_off[c] = lo;
    if (c == nc) continue;
    int64_t fr = 0, mt = 0;
    int y = INT_MIN;
    for (long long f = lo; f < n && D.fl_code[f] == c; ++f) {
      const unsigned long long kf = key[f];
      y = (int)((long long)kYBias - (long long)((kf >> 21) & ((1ull << 21) - 1)));
      const unsigned long long bk = kf & ((1ull << 21) - 1);
      D.fl_b[f] = bk == (1ull << 21) - 1 ? kFreeB : (int)bk;
      D.fl_cnt[f] = val[f];
      D.fl_pre[f] = mt;
      if (bk == (1ull << 21) - 1) fr += val[f];
      else mt += val[f];
    }
    D.dy[c] = y;
    D.dfree[c] = fr;
    D.dmatched[c] = mt;
    D.consumed[c] = 0;
  }
}
__global__ void ot_rebuild_kernel(OtDev D, const unsigned long long* __restrict__ key,
                                  const int64_t* __restrict__ val, long long n) {
  ot_rebuild_body(D, key, val, n, blockIdx.x, gridDim.x);
}

// ---- device-sized phase helpers ----------------------------------------------
// adm_off = exclusive prefix of adm_len[0, nf), adm_off[nf] = total: one
// block (n_free <= n_b), each thread a contiguous chunk.
__device__ __forceinline__ void ot_adm_scan_body(OtDev& D, int bid, int nb) {
  if (ot_hold(D)) return;
  const int nf = (int)D.ctr[kCtrFree];
  const int per = (nf + blockDim.x - 1) / blockDim.x;
  const int lo = min(nf, (int)threadIdx.x * per), hi = min(nf, lo + per);
  int64_t sum = 0;
  for (int i = lo; i < hi; ++i) sum += D.adm_len[i];
  __shared__ int64_t s_part[1024];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive (Hillis-Steele)
    const int64_t y = (int)threadIdx.x >= o ? s_part[threadIdx.x - o] : 0;
    __syncthreads();
    s_part[threadIdx.x] += y;
    __syncthreads();
  }
  int64_t run = s_part[threadIdx.x] - sum;
  for (int i = lo; i < hi; ++i) {
    D.adm_off[i] = run;
    run += D.adm_len[i];
  }
  if (threadIdx.x == blockDim.x - 1) D.adm_off[nf] = s_part[threadIdx.x];
}
__global__ void __launch_bounds__(1024) ot_adm_scan_kernel(OtDev D) { ot_adm_scan_body(D, blockIdx.x, gridDim.x); }

// After the batch of claim rounds: not over (or a round that needs the sort)
// -> the host continues them.
__device__ __forceinline__ void ot_da_gate_body(OtDev& D, int bid, int nb) {
  if (!ot_hold(D) && D.ctr[kCtrDone] != 1) D.ctr[kCtrHold] = 2;
}
__global__ void ot_da_gate_kernel(OtDev D) { ot_da_gate_body(D, blockIdx.x, gridDim.x); }

// The records (keys, counts) of the next state sorted and merged in one block
// (bitonic sort of the next power of two in shared memory, then one thread
// per run of equal keys), written back over the input; ctr[kCtrNFlows] =
// runs.  More than kOtSmallRec records: kCtrHold = 3 (the host sorts).
__device__ __forceinline__ void ot_small_merge_body(OtDev& D, unsigned long long* __restrict__ key,
                                                             int64_t* __restrict__ val, int bid, int nb) {
  if (ot_hold(D)) return;
  const int n = (int)D.ctr[kCtrRec];
  if (n > kOtSmallRec) {
    if (threadIdx.x == 0) D.ctr[kCtrHold] = 3;
    return;
  }
  extern __shared__ __align__(16) unsigned long long s_key[];
  int P = 2;
  while (P < n) P <<= 1;
  int64_t* s_val = reinterpret_cast<int64_t*>(s_key + P);
  __shared__ int s_heads[1024];
  if (max(P, 32) <= (int)blockDim.x) {
    // One element per thread: the bitonic network in registers, strides
    // below 32 by warp shuffles (no block barrier), larger ones through
    // shared memory; then the runs by a warp-shuffle block scan.
    const int P32 = max(P, 32), t = threadIdx.x, lane = t & 31, wid = t >> 5;
    s_val = reinterpret_cast<int64_t*>(s_key + P32);
    unsigned long long kk = t < n ? key[t] : ~0ull;
    int64_t vv = t < n ? val[t] : 0;
    for (int k = 2; k <= P32; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        unsigned long long kp = 0ull;
        int64_t vp = 0;
        if (j >= 32) {
          __syncthreads();
          if (t < P32) {
            s_key[t] = kk;
            s_val[t] = vv;
          }
          __syncthreads();
          if (t < P32) {
            kp = s_key[t ^ j];
            vp = s_val[t ^ j];
          }
        } else if (t < P32) {  // (whole warps: P32 is a multiple of 32)
          kp = __shfl_xor_sync(kFull, kk, j);
          vp = __shfl_xor_sync(kFull, vv, j);
        }
        if (t < P32) {
          const bool up = (t & k) == 0, lower = (t & j) == 0;
          if (lower == up ? (kp < kk) : (kp > kk)) {  // the lower index keeps the min when ascending
            kk = kp;
            vv = vp;
          }
        }
      }
    __syncthreads();
    if (t < P32) {
      s_key[t] = kk;
      s_val[t] = vv;
    }
    __syncthreads();
    const int hd = (t < n && (t == 0 || s_key[t] != s_key[t - 1])) ? 1 : 0;
    int inc = hd;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_heads[wid] = inc;
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < wid) before += s_heads[w];
      total += s_heads[w];
    }
    if (hd) {
      int64_t sum = 0;
      for (int q = t; q < n && s_key[q] == kk; ++q) sum += s_val[q];
      const int out = before + inc - 1;
      key[out] = kk;
      val[out] = sum;
    }
    if (t == 0) D.ctr[kCtrNFlows] = total;
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    s_key[i] = i < n ? key[i] : ~0ull;
    s_val[i] = i < n ? val[i] : 0;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long ki = s_key[i], kl = s_key[l];
          if (((i & k) == 0) == (ki > kl)) {
            s_key[i] = kl;
            s_key[l] = ki;
            const int64_t t = s_val[i];
            s_val[i] = s_val[l];
            s_val[l] = t;
          }
        }
      }
      __syncthreads();
    }
  // runs: thread chunks of the sorted keys, heads counted per chunk, scanned
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int h = 0;
  for (int i = lo; i < hi; ++i) h += (i == 0 || s_key[i] != s_key[i - 1]);
  s_heads[threadIdx.x] = h;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int y = (int)threadIdx.x >= o ? s_heads[threadIdx.x - o] : 0;
    __syncthreads();
    s_heads[threadIdx.x] += y;
    __syncthreads();
  }
  int out = s_heads[threadIdx.x] - h;
  for (int i = lo; i < hi; ++i) {
    if (i != 0 && s_key[i] == s_key[i - 1]) continue;
    int64_t sum = 0;
    for (int q = i; q < n && s_key[q] == s_key[i]; ++q) sum += s_val[q];
    key[out] = s_key[i];
    val[out] = sum;
    ++out;
  }
  if (threadIdx.x == blockDim.x - 1) D.ctr[kCtrNFlows] = s_heads[threadIdx.x];
}
__global__ void __launch_bounds__(1024) ot_small_merge_kernel(OtDev D, unsigned long long* __restrict__ key,
                                                             int64_t* __restrict__ val) {
  ot_small_merge_body(D, key, val, blockIdx.x, gridDim.x);
}



// ---- record merge beyond one block: buckets per demand vertex ------------------
// (persistent loop, n_rec > kOtSmallRec) records counted per vertex a (da_cnt,
// zero outside the claim rounds), bucket offsets by one block (da_off), the
// records scattered into their buckets (r_key2 / r_val2, da_fill), then a warp
// per vertex ranks its bucket (keys within one a differ in (y, b)), merges
// equal keys into the first of them and writes the unique records sorted at
// the bucket start, the unique counts scanned again, and the buckets copied
// compactly to key / val: the CUB sort + reduce-by-key result.  A bucket of
// more than kOtBucketMax records holds (3) for the host sort.
constexpr int kOtBucketMax = 1024;

__device__ __forceinline__ int ot_rec_a(unsigned long long k) { return (int)(k >> 42); }

__device__ __forceinline__ void ot_bucket_count_body(OtDev& D, const unsigned long long* key, int bid, int nb) {
  const long long n = D.ctr[kCtrRec];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x)
    atomicAdd(&D.da_cnt[ot_rec_a(key[j])], 1);
}

// one block: da_off[a] = exclusive prefix of cnt[0, n_a); a bucket past the
// cap sets the hold
__device__ __forceinline__ void ot_bucket_scan_body(OtDev& D, const int32_t* cnt, int64_t* off, int64_t* total) {
  const int n = D.n_a;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int64_t sum = 0;
  bool big = false;
  for (int i = lo; i < hi; ++i) {
    sum += cnt[i];
    big |= cnt[i] > kOtBucketMax;
  }
  __shared__ int64_t s_p[1024];
  s_p[threadIdx.x] = sum;
  if (big) D.ctr[kCtrHold] = 3;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const int64_t y = (int)threadIdx.x >= o ? s_p[threadIdx.x - o] : 0;
    __syncthreads();
    s_p[threadIdx.x] += y;
    __syncthreads();
  }
  int64_t run = s_p[threadIdx.x] - sum;
  for (int i = lo; i < hi; ++i) {
    off[i] = run;
    run += cnt[i];
  }
  if (threadIdx.x == blockDim.x - 1 && total) *total = s_p[threadIdx.x];
  __syncthreads();
}

__device__ __forceinline__ void ot_bucket_scatter_body(OtDev& D, const unsigned long long* key, const int64_t* val,
                                                       int bid, int nb) {
  const long long n = D.ctr[kCtrRec];
  for (long long j = bid * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)nb * blockDim.x) {
    const unsigned long long k = key[j];
    const int a = ot_rec_a(k);
    const long long pos = D.da_off[a] + atomicAdd(&D.da_fill[a], 1);
    D.r_key2[pos] = k;
    D.r_val2[pos] = val[j];
  }
}

// warp per vertex: unique keys sorted at the bucket start, da_cnt[a] = their
// count.  Lane-held chunks of the bucket: pass 1 gives every entry its run's
// sum and whether it is the first of its run; pass 2 counts the first entries
// with smaller keys (the entry's slot among the unique keys); the first
// entries then write their run in place (every read is done by then).
__device__ __forceinline__ void ot_bucket_merge_body(OtDev& D, int bid, int nb) {
  constexpr int kCh = kOtBucketMax / 32;
  const int lane = threadIdx.x & 31;
  const int warps = nb * (blockDim.x >> 5);
  for (int a = bid * (blockDim.x >> 5) + (threadIdx.x >> 5); a < D.n_a; a += warps) {
    const int c = D.da_cnt[a];
    if (c == 0) continue;
    const long long o = D.da_off[a];
    unsigned long long* k = D.r_key2 + o;
    int64_t* v = D.r_val2 + o;
    const int chunks = (c + 31) >> 5;
    unsigned long long hk[kCh];
    int64_t hs[kCh];
    bool first[kCh];
    int rank[kCh];
#pragma unroll 1
    for (int q = 0; q < chunks; ++q) {
      const int e = q * 32 + lane;
      const unsigned long long ke = e < c ? k[e] : ~0ull;
      int64_t sum = 0;
      bool f = e < c;
#pragma unroll 1
      for (int b1 = 0; b1 < c; b1 += 32) {
        const int e2 = b1 + lane;
        const unsigned long long k2 = e2 < c ? k[e2] : ~0ull;
        const int64_t v2 = e2 < c ? v[e2] : 0;
        const int m = min(32, c - b1);
        for (int t = 0; t < m; ++t) {
          const unsigned long long kt = __shfl_sync(kFull, k2, t);
          const int64_t vt = __shfl_sync(kFull, v2, t);
          if (kt == ke) {
            sum += vt;
            if (b1 + t < e) f = false;
          }
        }
      }
      hk[q] = ke;
      hs[q] = sum;
      first[q] = f;
      rank[q] = 0;
    }
#pragma unroll 1
    for (int q2 = 0; q2 < chunks; ++q2) {
      const unsigned long long kq = hk[q2];
      const int fq = first[q2] ? 1 : 0;
      const int m = min(32, c - q2 * 32);
      for (int t = 0; t < m; ++t) {
        const unsigned long long kt = __shfl_sync(kFull, kq, t);
        if (__shfl_sync(kFull, fq, t))
          for (int q = 0; q < chunks; ++q) rank[q] += kt < hk[q];
      }
    }
    int uniq = 0;
    for (int q = 0; q < chunks; ++q) uniq += __popc(__ballot_sync(kFull, first[q]));
    __syncwarp();
    for (int q = 0; q < chunks; ++q)
      if (first[q]) {
        k[rank[q]] = hk[q];
        v[rank[q]] = hs[q];
      }
    if (lane == 0) D.da_cnt[a] = uniq;
  }
}

// the unique runs of every bucket to key / val, compact and in vertex order
// (rec_off: the scan of the unique counts); the bucket counters back to zero
__device__ __forceinline__ void ot_bucket_copy_body(OtDev& D, unsigned long long* key, int64_t* val, int bid,
                                                    int nb) {
  const int lane = threadIdx.x & 31;
  const int warps = nb * (blockDim.x >> 5);
  for (int a = bid * (blockDim.x >> 5) + (threadIdx.x >> 5); a < D.n_a; a += warps) {
    const int u = D.da_cnt[a];
    const long long src = D.da_off[a], dst = D.rec_off[a];
    for (int j = lane; j < u; j += 32) {
      key[dst + j] = D.r_key2[src + j];
      val[dst + j] = D.r_val2[src + j];
    }
    __syncwarp();
    if (lane == 0) {
      D.da_cnt[a] = 0;
      D.da_fill[a] = 0;
    }
  }
}

// ---- the persistent phase loop (one cooperative launch) --------------------------
__device__ __forceinline__ void ot_grid_bar(OtDev& D, unsigned& target, int nb) {
  if (nb == 1) {  // one block: the block barrier is the grid barrier
    __syncthreads();
    return;
  }
  target += (unsigned)nb;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(D.bar) : "memory");
    if ((int)(ld_acquire(D.bar) - target) < 0) {
      const unsigned long long t0 = globaltimer();
      while ((int)(ld_acquire(D.bar) - target) < 0) {
        if (globaltimer() - t0 > 4000000000ull) {
          ot_fail(D, 6, (int)blockIdx.x);
          break;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t ot_vol(const int64_t* p) { return *(volatile const int64_t*)p; }

template <typename T>
__global__ void __launch_bounds__(1024, 1) ot_phase_loop_kernel(OtDev D, int stage, double threshold, int* counts) {
  const int bid = blockIdx.x, nb = gridDim.x;
  const bool lead = bid == 0 && threadIdx.x == 0;
  unsigned target = *(volatile unsigned*)(D.bar + 1);
  int64_t* ctr = D.ctr;
  D.in_loop = 1;
  // (optional per-step timeline: block 0's time from the previous barrier to
  // the end of barrier k, summed over the launch into D.steptime[k])
  unsigned long long t_prev = (D.steptime && lead) ? globaltimer() : 0ull;
#define OT_BAR(k)                                                   \
  do {                                                              \
    ot_grid_bar(D, target, nb);                                     \
    if (D.steptime && lead) {                                       \
      const unsigned long long now_ = globaltimer();                \
      D.steptime[k] += now_ - t_prev;                               \
      t_prev = now_;                                                \
    }                                                               \
  } while (0)
  while (true) {
    if (stage <= 0) {
      const int64_t n_i = ot_vol(ctr + kCtrNi);
      if ((double)n_i <= threshold || ot_vol(D.loop) >= D.fc_cap || *(volatile int*)D.status != 0) {
        if (lead) ctr[kCtrHold] = *(volatile int*)D.status != 0 ? 11 : ((double)n_i <= threshold ? 9 : 10);
        break;
      }
      if (lead) {
        for (int k = 2; k < kCtrCount; ++k) ctr[k] = 0;
        D.fcounts[D.loop[0]] = n_i;
      }
      OT_BAR(1);
      ot_t_body<T>(D, bid, nb);
      OT_BAR(2);
      ot_adm_body<T, 0>(D, bid, nb);
      OT_BAR(3);
      if (bid == 0) ot_adm_scan_body(D, bid, 1);
      OT_BAR(4);
    }
    if (stage <= 1) {
      const int nf = (int)ot_vol(ctr + kCtrFree);
      const int64_t total = ot_vol(D.adm_off + nf);
      if (total > D.adm_cap || total + nf + 1 > D.e_cap) {  // (uniform: every block reads the same)
        if (lead) ctr[kCtrHold] = 1;
        break;
      }
      ot_adm_body<T, 1>(D, bid, nb);
      ot_cut_init_body(D, bid, nb);
      OT_BAR(5);
    }
    if (stage <= 2) {
      bool big = false;
      while (true) {
        ot_da_propose_batched_body(D, bid, nb);
        OT_BAR(6);
        ot_da_count_body(D, bid, nb);
        OT_BAR(7);
        if (ot_vol(ctr + kCtrDone) != 0) break;
        ot_da_alloc_body(D, bid, nb);
        OT_BAR(8);
        ot_da_scatter_body(D, bid, nb);
        OT_BAR(9);
        if (ot_vol(ctr + kCtrDone) == 2) {
          big = true;
          break;
        }
        ot_da_resolve_warp_body(D, bid, nb);
        OT_BAR(10);
      }
      if (big) {  // a cluster past the warp resolve: that round sorted on the host
        if (lead) ctr[kCtrHold] = 2;
        break;
      }
    }
    if (stage <= 3) {
      if (ot_vol(D.fl_off + 2 * D.n_a) + ot_vol(ctr + kCtrE) + 2 * (int64_t)D.n_a + 16 > D.r_cap) {
        if (lead) ctr[kCtrHold] = 4;
        break;
      }
      ot_consumed_body(D, D.e_key, D.e_val, -1, bid, nb);
      ot_claim_records_body(D, D.e_key, D.e_val, -1, bid, nb);
      OT_BAR(11);
      ot_flow_records_body<T>(D, bid, nb);
      OT_BAR(12);
      ot_supply_body(D, bid, nb);
      if (ot_vol(ctr + kCtrRec) <= min(D.small_rec, kOtSmallRec)) {  // one block: bitonic sort + merge
        if (bid == 0) {
          __syncthreads();  // (block 0's supply threads done; the merge needs the whole block)
          ot_small_merge_body(D, D.r_key, D.r_val, bid, 1);
        }
        OT_BAR(13);
      } else {  // buckets per demand vertex (the r_key2 / r_val2 scratch, da_cnt / da_fill / da_off)
        ot_bucket_count_body(D, D.r_key, bid, nb);
        OT_BAR(14);
        if (bid == 0) ot_bucket_scan_body(D, D.da_cnt, D.da_off, nullptr);
        OT_BAR(15);
        if (ot_vol(ctr + kCtrHold) != 0) {  // a bucket past the cap: counters back to zero, host sort
          for (int a = bid * blockDim.x + threadIdx.x; a < D.n_a; a += nb * blockDim.x) D.da_cnt[a] = 0;
          OT_BAR(16);
          break;
        }
        ot_bucket_scatter_body(D, D.r_key, D.r_val, bid, nb);
        OT_BAR(17);
        ot_bucket_merge_body(D, bid, nb);
        OT_BAR(18);
        if (bid == 0) ot_bucket_scan_body(D, D.da_cnt, D.rec_off, ctr + kCtrNFlows);
        OT_BAR(19);
        ot_bucket_copy_body(D, D.r_key, D.r_val, bid, nb);
        OT_BAR(20);
      }
      if (ot_vol(ctr + kCtrHold) != 0) break;  // 3: more records than one block merges
    }
    ot_slot_body(D, D.r_key, -1, bid, nb);
    OT_BAR(21);
    ot_rebuild_body(D, D.r_key, D.r_val, -1, bid, nb);
    if (lead) {
      ctr[kCtrNi] = 0;
      D.loop[0] += 1;
      D.loop[1] += ctr[kCtrRounds];
    }
    OT_BAR(22);
    ot_free_count_body(D, counts, bid, nb);
    OT_BAR(23);
    ot_free_write_body(D, counts, bid, nb);
    OT_BAR(24);
    stage = 0;
  }
#undef OT_BAR
  if (lead) D.bar[1] = target;
}

}  // namespace

cudaError_t ot_dev_free_list(OtDev& D, int* scratch, cudaStream_t s) {
  ot_free_count_kernel<<<kListBlocks, 1024, 0, s>>>(D, scratch);
  ot_free_write_kernel<<<kListBlocks, 1024, 0, s>>>(D, scratch);
  return cudaGetLastError();
}

cudaError_t ot_dev_t(OtDev& D, cudaStream_t s) {
  with_width(D.width, [&](auto tag) {
    ot_t_kernel<decltype(tag)><<<148, 256, 0, s>>>(D);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t ot_dev_adm(OtDev& D, int pass, cudaStream_t s) {
  with_width(D.width, [&](auto tag) {
    if (pass == 0) ot_adm_kernel<decltype(tag), 0><<<148 * 8, 256, 0, s>>>(D);
    else ot_adm_kernel<decltype(tag), 1><<<148 * 8, 256, 0, s>>>(D);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t ot_dev_cut_init(OtDev& D, cudaStream_t s) {
  ot_cut_init_kernel<<<(2 * D.n_a + 255) / 256, 256, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_propose(OtDev& D, cudaStream_t s) {
  ot_da_propose_kernel<<<148 * 4, 256, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_da_rounds(OtDev& D, int rounds, cudaStream_t s) {
  for (int r = 0; r < rounds; ++r) {
    ot_da_propose_batched_kernel<<<148 * 2, 256, 0, s>>>(D);
    ot_da_count_kernel<<<148 * 2, 256, 0, s>>>(D);
    ot_da_alloc_kernel<<<148, 256, 0, s>>>(D);
    ot_da_scatter_kernel<<<148 * 2, 256, 0, s>>>(D);
    ot_da_resolve_warp_kernel<<<148 * 8, 256, 0, s>>>(D);
  }
  return cudaGetLastError();
}

cudaError_t ot_dev_phase_begin(OtDev& D, cudaStream_t s) {
  return cudaMemsetAsync(D.ctr + 2, 0, (kCtrCount - 2) * sizeof(int64_t), s);
}

cudaError_t ot_dev_adm_scan(OtDev& D, cudaStream_t s) {
  ot_adm_scan_kernel<<<1, 1024, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_da_gate(OtDev& D, cudaStream_t s) {
  ot_da_gate_kernel<<<1, 1, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_small_merge(OtDev& D, unsigned long long* key, int64_t* val, cudaStream_t s) {
  const size_t smem = (size_t)kOtSmallRec * 16;
  smem_attr_raise(reinterpret_cast<const void*>(ot_small_merge_kernel), smem);
  ot_small_merge_kernel<<<1, 1024, smem, s>>>(D, key, val);
  return cudaGetLastError();
}

cudaError_t ot_dev_phase_loop(OtDev& D, int stage, double threshold, int* scratch, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  with_width(D.width, [&](auto tag) {
    using T = decltype(tag);
    auto fn = ot_phase_loop_kernel<T>;
    const size_t smem = (size_t)kOtSmallRec * 16;
    smem_attr_raise(reinterpret_cast<const void*>(fn), smem);
    int dev = 0, sms = 148, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 1024, smem) != cudaSuccess || per < 1) {
      e = cudaErrorLaunchOutOfResources;
      return 0;
    }
    // blocks: one per 64 supply vertices up to one per SM (small instances
    // are barrier-bound: fewer blocks, cheaper barriers; one block needs none)
    const int grid = std::max(1, std::min(std::min(sms, kListBlocks), D.n_b / 64));
    void* args[] = {&D, &stage, &threshold, &scratch};
    // threads per block: 1024 for few blocks (the one-block merges dominate),
    // 512 from 32 blocks on (scripts/ab_ot_threads.sh: n = 5k / 20k -15 / -7 %,
    // n = 1k +4 %); OTPRG_OT_THREADS overrides (A/B)
    static const int forced = [] {
      const char* v = std::getenv("OTPRG_OT_THREADS");
      const int t = v ? std::atoi(v) : 0;
      return t >= 128 && t <= 1024 && t % 32 == 0 ? t : 0;
    }();
    const int threads = forced ? forced : (grid >= 32 ? 512 : 1024);
    e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(threads), args, smem, s);
    return 0;
  });
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t ot_dev_da_clear(OtDev& D, cudaStream_t s) {
  ot_da_clear_kernel<<<148, 256, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_resolve(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           unsigned long long* out_key, int64_t* out_val, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  ot_da_resolve_kernel<<<(int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(D, key, val, n, out_key,
                                                                                          out_val);
  return cudaGetLastError();
}

cudaError_t ot_dev_consumed(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                            cudaStream_t s) {
  if (n != 0)
    ot_consumed_kernel<<<n < 0 ? 148 * 4 : (int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(D, key,
                                                                                                       val, n);
  return cudaGetLastError();
}

cudaError_t ot_dev_records(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           cudaStream_t s) {
  with_width(D.width, [&](auto tag) {
    ot_flow_records_kernel<decltype(tag)><<<148 * 8, 256, 0, s>>>(D);
    return 0;
  });
  if (n != 0)
    ot_claim_records_kernel<<<n < 0 ? 148 * 4 : (int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
        D, key, val, n);
  ot_supply_kernel<<<(D.n_b + 255) / 256, 256, 0, s>>>(D);
  return cudaGetLastError();
}

cudaError_t ot_dev_rebuild(OtDev& D, const unsigned long long* key, const int64_t* val, long long n,
                           cudaStream_t s) {
  if (n != 0)
    ot_slot_kernel<<<n < 0 ? 148 * 4 : (int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(D, key, n);
  ot_rebuild_kernel<<<(2 * D.n_a + 1 + 255) / 256, 256, 0, s>>>(D, key, val, n);
  return cudaGetLastError();
}

// CUB helpers (temp storage grown on demand by the caller).
cudaError_t ot_sort_pairs(void* temp, size_t& temp_bytes, const unsigned long long* kin, unsigned long long* kout,
                          const int64_t* vin, int64_t* vout, long long n, int end_bit, cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kin, kout, vin, vout, n, 0, end_bit, s);
}

cudaError_t ot_reduce_by_key(void* temp, size_t& temp_bytes, const unsigned long long* kin,
                             unsigned long long* kout, const int64_t* vin, int64_t* vout, long long* nout,
                             long long n, cudaStream_t s) {
  return cub::DeviceReduce::ReduceByKey(temp, temp_bytes, kin, kout, vin, vout, nout, cub::Sum(), n, s);
}

cudaError_t ot_exclusive_sum(void* temp, size_t& temp_bytes, const int64_t* in, int64_t* out, int n,
                             cudaStream_t s) {
  return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n, s);
}

}  // namespace otprg
