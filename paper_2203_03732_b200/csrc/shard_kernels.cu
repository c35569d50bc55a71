// shard_kernels.cu — the A-row-sharded phase step for several GPUs
// (SURVEY §8(e)).  Shard g owns the demand range [lo_g, hi_g) of every kT
// row; the matching, duals and holders are replicated on every rank and every
// rank runs the same deterministic deferred acceptance, so all ranks hold the
// identical state after each phase and only candidate lists cross NVLink.
//
// Per phase (host-driven, one process per GPU; see shard_host in
// otprg_capi.cpp and paper_2203_03732_b200/sharded.py):
//   shard_top   apply M' of the previous phase (apply_phase,
//               assignment.cpp:210-235), termination / phase cap
//               (:324-334, :356-358), inverse map b -> list index;
//   shard_scan  every rank scans its slab of each free b's row for the first
//               K admissible a (global index) and its coverage end, into its
//               slot of the exchange buffer;
//   exchange    all-gather of the slots (NCCL over NVLink; nothing to do when
//               all shards share one buffer);
//   shard_da    deferred acceptance over the merged candidate lists (shards
//               are ascending ranges, so concatenation is ascending); a chain
//               that reaches a truncated shard's coverage end parks with a
//               restart position, the parked rows are rescanned and
//               exchanged, and the chains resume.  DA is order independent,
//               so the result is the reference's sequential greedy M'
//               whatever the shard count.
#include <algorithm>
#include <climits>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

#ifndef OTPRG_SHARD_UNROLL
#define OTPRG_SHARD_UNROLL 12  // A/B (scripts/ab_shard_unroll.sh): 4 / 8 / 12 / 16 / 24 -> 13.6 / 13.5 / 12.1 / 15.8 / 18.3 ms
#endif

__device__ __forceinline__ uint32_t t_get(const ShardArgs& S, int a) {
  return S.width == 1   ? (uint32_t)static_cast<const uint8_t*>(S.t)[a]
         : S.width == 2 ? (uint32_t)static_cast<const uint16_t*>(S.t)[a]
                        : static_cast<const uint32_t*>(S.t)[a];
}
__device__ __forceinline__ void t_set(const ShardArgs& S, int a, uint32_t v) {
  if (S.width == 1) static_cast<uint8_t*>(S.t)[a] = (uint8_t)v;
  else if (S.width == 2) static_cast<uint16_t*>(S.t)[a] = (uint16_t)v;
  else static_cast<uint32_t*>(S.t)[a] = v;
}

// Scan request: (list index, b, start position (global a)).  req == nullptr:
// every free b of the phase from position 0.
//
// segs == 1: one warp per request scans the slab row from `start` in 4 KB
// steps and writes the first K admissible a (ascending) and the resume
// position straight to the exchange slots.  segs > 1 (few requests, long
// rows: the tail phases): the row range [start, hi) is split into segs
// contiguous pieces, one warp each; every warp keeps the first K hits of its
// piece in S.seg_hits, and the last warp of the request to finish merges the
// pieces in order (the first K hits overall; resume after the K-th), so a
// 200 KB row costs a few dependent steps instead of ~50.
template <typename T, bool kP1>
__global__ void __launch_bounds__(256) shard_scan_kernel(ShardArgs S, const int4* __restrict__ req,
                                                         int nreq, int segs, int32_t* __restrict__ cand,
                                                         int2* __restrict__ meta) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  constexpr int kU = OTPRG_SHARD_UNROLL;  // 16-byte loads in flight per lane (12: 6 KB per warp step)
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nreq * segs) return;
  const int r = w / segs, sg = w - r * segs;
  int i, b, start;
  if (req) {
    const int4 q = req[r];
    i = q.x;
    b = q.y;
    start = q.z;
  } else {
    i = r;
    b = __ldcg(S.list_in + r);
    start = 0;
  }
  const uint32_t tg = SD::rep((uint32_t)__ldcg(S.yb + b) - 1u);
  const int lo = S.lo, hi = S.hi, K = S.K, width_local = hi - lo;
  int32_t* o = segs == 1 ? cand + ((size_t)S.shard * S.cap + i) * K : S.seg_hits + (size_t)w * K;
  int cnt = 0, cov = hi;
  const int lstart = max(start, lo) - lo;
  if (start < hi) {
    const uint4* rv = reinterpret_cast<const uint4*>(static_cast<const T*>(S.kT) + (size_t)b * S.lda);
    const uint4* tv = reinterpret_cast<const uint4*>(static_cast<const T*>(S.t) + lo);
    const int nv = (width_local + kEpv - 1) / kEpv;
    // this warp's piece, in 32-vector units
    const int u0 = (lstart / kEpv) >> 5, units = (nv + 31) >> 5;
    const int per = (units - u0 + segs - 1) / segs;
    const int vb = (u0 + sg * per) * 32, ve = min(nv, (u0 + (sg + 1) * per) * 32);
    bool full = false;
    for (int v = vb; v < ve && !full; v += 32 * kU) {
      uint4 kr[kU], tr[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int vi = v + j * 32 + lane;
        if (vi < ve) {
          kr[j] = __ldg(rv + vi);
          // phase 1: t == 0 everywhere (init_state), no t traffic
          tr[j] = kP1 ? make_uint4(0u, 0u, 0u, 0u) : __ldcg(tv + vi);
        } else {
          kr[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
          tr[j] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        if (full) break;
        const int e0 = (v + j * 32 + lane) * kEpv;  // local element index
        const uint32_t kw[4] = {kr[j].x, kr[j].y, kr[j].z, kr[j].w};
        const uint32_t tw[4] = {tr[j].x, tr[j].y, tr[j].z, tr[j].w};
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) m |= SD::bits(SD::eq(SD::add(kw[q], tw[q]), tg)) << (q * SD::kEpw);
        if (e0 < lstart) {
          const int drop = lstart - e0;
          m = drop >= kEpv ? 0u : (m & (~0u << drop));
        }
        if (e0 + kEpv > width_local) {  // t beyond the shard belongs to the next shard
          const int keepn = width_local - e0;
          m = keepn <= 0 ? 0u : (m & ((1u << keepn) - 1u));
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
        int idx = cnt + inc - c, last = -1;
        uint32_t bm = m;
        while (bm) {
          const int e = __ffs(bm) - 1;
          bm &= bm - 1;
          if (idx < K) {
            o[idx] = lo + e0 + e;
            if (idx == K - 1) last = lo + e0 + e;
          }
          ++idx;
        }
        if (cnt + tot >= K) {
          const unsigned src = __ballot_sync(kFull, last >= 0);
          cov = __shfl_sync(kFull, last, __ffs(src) - 1) + 1;
          cnt = K;
          full = true;
        } else {
          cnt += tot;
        }
      }
    }
  }
  if (segs == 1) {
    if (lane == 0) meta[(size_t)S.shard * S.cap + i] = make_int2(cnt, cov);
    return;
  }
  // publish this piece, then the request's last piece merges (first K overall)
  int prev = 0;
  if (lane == 0) {
    S.seg_cnt[w] = cnt;
    __threadfence();
    prev = atomicAdd(S.row_cnt + r, 1);
  }
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != segs - 1) return;
  __threadfence();
  int32_t* out = cand + ((size_t)S.shard * S.cap + i) * K;
  const int wb = r * segs;
  int tot = 0, rcov = hi;
  for (int p = 0; p < segs && tot < K; ++p) {
    const int c = __ldcg(S.seg_cnt + wb + p);
    const int32_t* src = S.seg_hits + (size_t)(wb + p) * K;
    if (lane < c && tot + lane < K) out[tot + lane] = __ldcg(src + lane);
    if (tot + c >= K) rcov = __ldcg(src + (K - 1 - tot)) + 1;
    tot = min(K, tot + c);
  }
  if (lane == 0) {
    meta[(size_t)S.shard * S.cap + i] = make_int2(tot, rcov);
    S.row_cnt[r] = 0;  // ready for the next launch
  }
}

// Top of the phase after `phase_done` phases: apply M' of phase phase_done
// (replicated), termination test, counters for the next phase.
__global__ void __launch_bounds__(1024) shard_top_kernel(ShardArgs S, uint32_t phase_done,
                                                         int apply, int cond) {
  Ctl* ctl = S.ctl;
  if (cond && ctl->work[1] != 0) return;  // chains parked: the phase goes on
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  const int par = phase_done & 1;
  if (apply) {
    const int m = ctl->mp_cnt[par];
    for (int q = gtid; q < m; q += gthreads) {
      const int2 e = S.mp_prev[q];
      const int a = e.x, old_b = e.y;
      const int b = (int)(uint32_t)S.holder[a];
      if (old_b >= 0) S.match_b[old_b] = -1;
      S.match_a[a] = b;
      S.match_b[b] = a;
      const uint32_t nt = t_get(S, a) + 1u;
      if (nt > ctl->tmax) report(ctl, 12, (int)phase_done, a, (int)nt);
      t_set(S, a, nt);
    }
  }
  const int n = ctl->cnt[par];
  if (gtid == 0) {
    ctl->phase = phase_done;
    if (apply) ctl->applied = phase_done;
    if (n <= ctl->thresh) {  // (double)n_i <= eps*m  <=>  n_i <= floor(eps*m)
      ctl->done = 1;
      ctl->full_match = (n == 0);
    } else if (phase_done + 1 > (uint32_t)ctl->phase_cap) {
      report(ctl, 5, (int)phase_done);
    } else {
      S.free_counts[phase_done] = n;
      ctl->sum_ni += n;
      const int nx = par ^ 1;  // counters the coming phase appends to
      ctl->cnt[nx] = 0;
      ctl->mp_cnt[nx] = 0;
      ctl->exh[nx] = 0;  // (work[1], the parked count, is reset before every DA launch)
    }
  }
}

// The free list of the coming phase, ascending b (identical on every rank,
// so list indices name the same b everywhere), and its inverse.  Two passes
// over kCompactBlocks contiguous ranges: per-range counts, then ordered writes
// at the range's offset (block-wide scans per 1024-entry tile).
constexpr int kCompactBlocks = 148;

__global__ void __launch_bounds__(1024) shard_compact_count_kernel(ShardArgs S, int cond, int* counts) {
  if (S.ctl->done || (cond && S.ctl->work[1] != 0)) return;
  const int n_b = S.ctl->n_b;
  const int chunk = (n_b + gridDim.x - 1) / gridDim.x;
  const int lo = min(n_b, (int)blockIdx.x * chunk), hi = min(n_b, lo + chunk);
  int c = 0;
  for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) c += (S.match_b[q] == -1);
  __shared__ int s_sum;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_sum, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_sum;
}

__global__ void __launch_bounds__(1024) shard_compact_write_kernel(ShardArgs S, int cond,
                                                                   const int* counts) {
  if (S.ctl->done || (cond && S.ctl->work[1] != 0)) return;
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int n_b = S.ctl->n_b;
  const int chunk = (n_b + gridDim.x - 1) / gridDim.x;
  const int lo = min(n_b, (int)blockIdx.x * chunk), hi = min(n_b, lo + chunk);
  if (threadIdx.x == 0) {
    int off = 0;
    for (int g = 0; g < (int)blockIdx.x; ++g) off += counts[g];
    s_base = off;
  }
  __syncthreads();
  int32_t* out = const_cast<int32_t*>(S.list_in);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int t0 = lo; t0 < hi; t0 += blockDim.x) {  // one tile: block-wide ordered scan of the flags
    const int q = t0 + threadIdx.x;
    const bool f = q < hi && S.match_b[q] == -1;
    const unsigned bal = __ballot_sync(kFull, f);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nwarps; ++w) {
      if (w < warp) before += s_warp[w];
      total += s_warp[w];
    }
    if (f) {
      const int pos = s_base + before + __popc(bal & ((1u << lane) - 1u));
      out[pos] = q;
      S.pos_of_b[q] = pos;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += total;
    __syncthreads();
  }
}

// Deferred acceptance over merged candidate lists, one warp per chain.
// resume_list == nullptr: a chain per free b; else per parked entry.
__global__ void __launch_bounds__(256) shard_da_kernel(ShardArgs S, uint32_t phase,
                                                       const int32_t* __restrict__ cand,
                                                       const int2* __restrict__ meta, int nchains,
                                                       const int4* __restrict__ resume_list) {
  Ctl* ctl = S.ctl;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nchains) return;
  const uint32_t cur_tag = ~phase;
  const int par = phase & 1;
  int i, b, start;
  if (resume_list) {
    const int4 r = resume_list[w];
    i = r.x;
    b = r.y;
    start = r.z;
  } else {
    i = w;
    b = __ldcg(S.list_in + w);
    start = 0;
  }
  const int K = S.K, G = S.n_shards;
  while (true) {
    int a = -1, restart = -1;
    for (int g = 0; g < G; ++g) {  // next candidate >= start, shard-ascending
      const int ghi = S.bounds[g + 1];
      if (start >= ghi) continue;
      const int2 mt = __ldcg(meta + (size_t)g * S.cap + i);
      int c = -1;
      if (lane < mt.x && lane < K) c = __ldcg(cand + ((size_t)g * S.cap + i) * K + lane);
      const unsigned bal = __ballot_sync(kFull, c >= start);
      if (bal) {
        a = __shfl_sync(kFull, c, __ffs(bal) - 1);
        break;
      }
      if (mt.y < ghi) {  // truncated shard: [max(start, cov), hi) not yet scanned
        restart = max(start, mt.y);
        break;
      }
    }
    if (a < 0 && restart >= 0) {  // park until the gap is rescanned
      if (lane == 0) {
        const int pos = atomicAdd(&ctl->work[1], 1);
        S.park_out[pos] = make_int4(i, b, restart, 0);
      }
      return;
    }
    if (a < 0) {  // b stays free: Y(b) += 1 (apply_phase :233-235)
      if (lane == 0) {
        const uint32_t yb = (uint32_t)__ldcg(S.yb + b);
        if (yb + 1 > ctl->tmax) report(ctl, 11, (int)phase, b, (int)yb);
        S.yb[b] = (int32_t)(yb + 1);
        atomicAdd(&ctl->cnt[par], 1);  // the next free list is rebuilt sorted
        atomicAdd(&ctl->exh[par], 1);
      }
      return;
    }
    const unsigned long long key = ((unsigned long long)cur_tag << 32) | (uint32_t)b;
    unsigned long long old = 0;
    if (lane == 0) old = atomicMin(S.holder + a, key);
    old = __shfl_sync(kFull, old, 0);
    if (old < key) {  // held by a lower b of this phase
      start = a + 1;
      continue;
    }
    if ((uint32_t)(old >> 32) == cur_tag) {  // displaced b2 continues after a
      b = (int)(uint32_t)old;
      i = __ldcg(S.pos_of_b + b);
      start = a + 1;
      continue;
    }
    if (lane == 0) {  // first holder this phase: the previous partner is freed
      const int partner = __ldcg(S.match_a + a);  // complete: applied at this phase's top
      if (partner >= 0) atomicAdd(&ctl->cnt[par], 1);
      const int pos = atomicAdd(&ctl->mp_cnt[par], 1);
      S.mp_out[pos] = make_int2(a, partner);
    }
    return;
  }
}


// On-the-fly variant (OTPRG_FLAG_ON_THE_FLY): no kT slab.  Each lane
// takes one demand point per 32-element group, forms d2 = dx*dx + dy*dy in
// IEEE round-to-nearest (the reference's bits, instances.cpp:70-75) and tests
// admissibility k(a,b) + t(a) == target as thr[m] <= d2 < thr[m+1] with
// m = target - t(a), against the exact threshold table staged in shared
// memory: no sqrt, no division, 16 B of point per element instead of w B of kT.
// Outputs, pieces and the merge as shard_scan_kernel.
template <typename T>
__global__ void __launch_bounds__(256) shard_scan_otf_kernel(ShardArgs S, const int4* __restrict__ req,
                                                             int nreq, int segs, int32_t* __restrict__ cand,
                                                             int2* __restrict__ meta) {
  extern __shared__ double s_thr[];
  for (int j = threadIdx.x; j < S.thr_n; j += blockDim.x) s_thr[j] = S.thr[j];
  __syncthreads();
  constexpr int kG = 8;  // 32-element groups per warp step
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nreq * segs) return;
  const int r = w / segs, sg = w - r * segs;
  int i, b, start;
  if (req) {
    const int4 q = req[r];
    i = q.x;
    b = q.y;
    start = q.z;
  } else {
    i = r;
    b = __ldcg(S.list_in + r);
    start = 0;
  }
  const int64_t target = (int64_t)(uint32_t)__ldcg(S.yb + b) - 1;
  const int lo = S.lo, hi = S.hi, K = S.K, width_local = hi - lo, mmax = S.thr_n - 2;
  int32_t* o = segs == 1 ? cand + ((size_t)S.shard * S.cap + i) * K : S.seg_hits + (size_t)w * K;
  int cnt = 0, cov = hi;
  const int lstart = max(start, lo) - lo;
  if (start < hi) {
    const double2 q = S.pb[b];
    const double2* pa = S.pa + lo;
    const T* tl = static_cast<const T*>(S.t) + lo;
    const int groups = (width_local + 31) >> 5, g0 = lstart >> 5;
    const int per = (groups - g0 + segs - 1) / segs;
    const int gb = g0 + sg * per, ge = min(groups, g0 + (sg + 1) * per);
    bool full = false;
    for (int g = gb; g < ge && !full; g += kG) {
      double2 p[kG];
      uint32_t tt[kG];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const int e = (g + j) * 32 + lane;
        const bool ok = g + j < ge && e < width_local;
        p[j] = ok ? __ldg(pa + e) : make_double2(0.0, 0.0);
        tt[j] = ok ? (uint32_t)__ldcg(tl + e) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        if (full || g + j >= ge) break;
        const int e = (g + j) * 32 + lane;
        bool hit = false;
        if (e < width_local && e >= lstart) {
          const double dx = __dsub_rn(p[j].x, q.x), dy = __dsub_rn(p[j].y, q.y);
          const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
          const int64_t m = target - (int64_t)tt[j];
          hit = m >= 0 && m <= mmax && s_thr[m] <= d2 && d2 < s_thr[m + 1];
        }
        const unsigned bal = __ballot_sync(kFull, hit);
        if (!bal) continue;
        const int idx = cnt + __popc(bal & ((1u << lane) - 1u));
        if (hit && idx < K) o[idx] = lo + e;
        const int c = __popc(bal);
        if (cnt + c >= K) {
          unsigned bm = bal;  // lane of the K-th hit overall: the (K - cnt)-th set bit
          for (int t2 = 1; t2 < K - cnt; ++t2) bm &= bm - 1;
          const int src = __ffs(bm) - 1;
          cov = lo + (g + j) * 32 + src + 1;
          cnt = K;
          full = true;
        } else {
          cnt += c;
        }
      }
    }
  }
  if (segs == 1) {
    if (lane == 0) meta[(size_t)S.shard * S.cap + i] = make_int2(cnt, cov);
    return;
  }
  int prev = 0;
  if (lane == 0) {
    S.seg_cnt[w] = cnt;
    __threadfence();
    prev = atomicAdd(S.row_cnt + r, 1);
  }
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != segs - 1) return;
  __threadfence();
  int32_t* out = cand + ((size_t)S.shard * S.cap + i) * K;
  const int wb = r * segs;
  int tot = 0, rcov = hi;
  for (int pc = 0; pc < segs && tot < K; ++pc) {
    const int c = __ldcg(S.seg_cnt + wb + pc);
    const int32_t* src = S.seg_hits + (size_t)(wb + pc) * K;
    if (lane < c && tot + lane < K) out[tot + lane] = __ldcg(src + lane);
    if (tot + c >= K) rcov = __ldcg(src + (K - 1 - tot)) + 1;
    tot = min(K, tot + c);
  }
  if (lane == 0) {
    meta[(size_t)S.shard * S.cap + i] = make_int2(tot, rcov);
    S.row_cnt[r] = 0;
  }
}


// On-the-fly, many requests: a block takes kOtfRows requests (one warp
// each) and streams the slab's demand points and t through shared memory in
// kOtfChunk-point chunks (two stages filled by 1-D TMA bulk copies, the next
// chunk landing while the current one is scanned), so each 16-byte point
// leaves L2 once per block rather than once per row; warps whose row already
// has K hits idle until every row of the block is done.  segs > 1 (tail
// phases: few row groups) splits the chunk range of a row group into pieces
// on separate blocks, merged per row like shard_scan_kernel's pieces.  The
// threshold table is staged as pairs (thr[m], thr[m+1]): one 16-byte load.
#ifndef OTPRG_OTF_ROWS
#define OTPRG_OTF_ROWS 16
#endif
#ifndef OTPRG_OTF_GU
#define OTPRG_OTF_GU 4
#endif
#ifndef OTPRG_OTF_CHUNK
#define OTPRG_OTF_CHUNK 2048
#endif
constexpr int kOtfRows = OTPRG_OTF_ROWS, kOtfChunk = OTPRG_OTF_CHUNK;

template <typename T, bool kP1>
__global__ void __launch_bounds__(kOtfRows * 32) shard_scan_otf_tiled_kernel(ShardArgs S,
                                                                            const int4* __restrict__ req,
                                                                            int nreq, int segs,
                                                                            int32_t* __restrict__ cand,
                                                                            int2* __restrict__ meta) {
  extern __shared__ __align__(128) unsigned char s_dyn[];
  // stage st: points [kOtfChunk] double2 then t [kOtfChunk] T; the pair table after both stages
  constexpr size_t kStage = (size_t)kOtfChunk * (sizeof(double2) + sizeof(T));
  double2* s_pair = reinterpret_cast<double2*>(s_dyn + 2 * kStage);
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ int s_lo_start, s_act[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = blockIdx.x / segs, sg = blockIdx.x - grp * segs;
  const int r = grp * kOtfRows + warp;
  const bool has = r < nreq;
  int i = 0, b = 0, start = 0;
  if (has) {
    if (req) {
      const int4 q = req[r];
      i = q.x;
      b = q.y;
      start = q.z;
    } else {
      i = r;
      b = __ldcg(S.list_in + r);
    }
  }
  const int lo = S.lo, hi = S.hi, K = S.K, width_local = hi - lo;
  const unsigned mmax = (unsigned)(S.thr_n - 2);
  const int lstart = has ? max(start, lo) - lo : width_local;
  bool done = !has || start >= hi;
  if (threadIdx.x == 0) {
    s_lo_start = width_local;
    s_act[0] = s_act[1] = s_act[2] = 0;
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j + 1 < S.thr_n; j += blockDim.x) s_pair[j] = make_double2(S.thr[j], S.thr[j + 1]);
  __syncthreads();
  if (lane == 0 && !done) atomicMin(&s_lo_start, lstart);
  int target = 0;  // (the table has <= 8192 levels: int is exact)
  double2 q = make_double2(0.0, 0.0);
  if (has) {
    target = __ldcg(S.yb + b) - 1;
    q = S.pb[b];
  }
  int32_t* o = segs == 1 ? cand + ((size_t)S.shard * S.cap + i) * K : S.seg_hits + ((size_t)r * segs + sg) * K;
  int cnt = 0, cov = hi;
  __syncthreads();
  // this block's piece of the row group's chunk range
  const int c_first = s_lo_start / kOtfChunk, c_total = (width_local + kOtfChunk - 1) / kOtfChunk;
  const int per = c_total > c_first ? (c_total - c_first + segs - 1) / segs : 0;
  const int k_lo = c_first + sg * per, k_hi = min(c_total, c_first + (sg + 1) * per);
  const int nchunk = max(0, k_hi - k_lo);
  const double2* pa = S.pa + lo;
  const T* tl = static_cast<const T*>(S.t) + lo;
  auto issue = [&](int k) {  // thread 0: chunk k_lo + k into stage k & 1
    const int c0 = (k_lo + k) * kOtfChunk;
    const int len = min(kOtfChunk, width_local - c0);
    unsigned char* st = s_dyn + (size_t)(k & 1) * kStage;
    const unsigned pb_bytes = (unsigned)len * 16u;
    const unsigned tb = (unsigned)(((size_t)len * sizeof(T) + 15) & ~(size_t)15);
    mbar_expect_tx(&bar[k & 1], pb_bytes + (kP1 ? 0u : tb));
    bulk_g2s(st, pa + c0, pb_bytes, &bar[k & 1]);
    if (!kP1) bulk_g2s(st + (size_t)kOtfChunk * sizeof(double2), tl + c0, tb, &bar[k & 1]);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < min(2, nchunk); ++k) issue(k);
  unsigned par = 0;
  int k = 0;
  for (; k < nchunk; ++k) {
    mbar_wait(&bar[k & 1], (par >> (k & 1)) & 1u);
    par ^= 1u << (k & 1);
    const int c0 = (k_lo + k) * kOtfChunk;
    const int len = min(kOtfChunk, width_local - c0);
    const double2* sp = reinterpret_cast<const double2*>(s_dyn + (size_t)(k & 1) * kStage);
    const T* stt = reinterpret_cast<const T*>(s_dyn + (size_t)(k & 1) * kStage + (size_t)kOtfChunk * sizeof(double2));
    // steps of 32 * kGU elements from a multiple of 32 * kGU (elements
    // before lstart are masked), so every index stays inside the stage
    const double thr1 = s_pair[0].y;
    const int g_begin = max(0, ((lstart - c0) / (32 * OTPRG_OTF_GU)) * (32 * OTPRG_OTF_GU));
    auto test = [&](int g) -> bool {  // is element c0 + g + lane admissible?
      // branch-free: the kernel is issue-bound, and an early return costs a
      // reconvergence region (BSSY/BSYNC + a divergence check) per element;
      // out-of-range lanes compute on stale stage data and are masked
      const int e = g + lane;
      const double2 p = sp[e];
      const double dx = __dsub_rn(p.x, q.x), dy = __dsub_rn(p.y, q.y);
      const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      if constexpr (kP1) {  // phase 1: t == 0 and target == 0, so level 0: d2 < thr[1]
        return (e < len) & (c0 + e >= lstart) & (d2 < thr1);
      } else {
        const unsigned m = (unsigned)(target - (int)stt[e]);
        const double2 tw = s_pair[min(m, mmax)];
        return (e < len) & (c0 + e >= lstart) & (m <= mmax) & (tw.x <= d2) & (d2 < tw.y);
      }
    };
    auto take = [&](int g, unsigned bal, bool hit) {  // append a group's hits in lane order
      const int idx = cnt + __popc(bal & ((1u << lane) - 1u));
      if (hit && idx < K) o[idx] = lo + c0 + g + lane;
      const int cc = __popc(bal);
      if (cnt + cc >= K) {
        unsigned bm = bal;
        for (int t2 = 1; t2 < K - cnt; ++t2) bm &= bm - 1;
        cov = lo + c0 + g + __ffs(bm);  // (position of the K-th hit) + 1
        cnt = K;
        done = true;
      } else {
        cnt += cc;
      }
    };
    constexpr int kGU = OTPRG_OTF_GU;  // groups per step (independent loads and DP ops in flight)
    for (int g = g_begin; g < len && !done; g += 32 * kGU) {
      bool h[kGU];
      unsigned bl[kGU], any = 0;
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        h[u] = test(g + 32 * u);
        bl[u] = __ballot_sync(kFull, h[u]);
        any |= bl[u];
      }
      if (!any) continue;
#pragma unroll
      for (int u = 0; u < kGU; ++u)
        if (bl[u] && !done) take(g + 32 * u, bl[u], h[u]);
    }
    // rows still open after this chunk; three counters so that a reset never
    // races with a read (counter k % 3 is read after this barrier, reset after
    // the next one, and counted into again only after the one after that)
    if (lane == 0 && !done) atomicAdd(&s_act[k % 3], 1);
    __syncthreads();  // stage k & 1 consumed by every warp
    const int open = s_act[k % 3];
    if (threadIdx.x == 0) s_act[(k + 2) % 3] = 0;
    if (open == 0) {
      ++k;
      break;
    }
    if (threadIdx.x == 0 && k + 2 < nchunk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + 2);
    }
  }
  // an early stop leaves the chunk after the last consumed one in flight:
  // it must land before the block exits
  if (threadIdx.x == 0 && k < nchunk) mbar_wait(&bar[k & 1], (par >> (k & 1)) & 1u);
  if (!has) return;
  if (segs == 1) {
    if (lane == 0) meta[(size_t)S.shard * S.cap + i] = make_int2(cnt, cov);
    return;
  }
  // publish this piece; the row's last piece merges (first K overall)
  const int w = r * segs + sg;
  int prev = 0;
  if (lane == 0) {
    S.seg_cnt[w] = cnt;
    __threadfence();
    prev = atomicAdd(S.row_cnt + r, 1);
  }
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != segs - 1) return;
  __threadfence();
  int32_t* out = cand + ((size_t)S.shard * S.cap + i) * K;
  const int wb = r * segs;
  int tot = 0, rcov = hi;
  for (int pc = 0; pc < segs && tot < K; ++pc) {
    const int c = __ldcg(S.seg_cnt + wb + pc);
    const int32_t* src = S.seg_hits + (size_t)(wb + pc) * K;
    if (lane < c && tot + lane < K) out[tot + lane] = __ldcg(src + lane);
    if (tot + c >= K) rcov = __ldcg(src + (K - 1 - tot)) + 1;
    tot = min(K, tot + c);
  }
  if (lane == 0) {
    meta[(size_t)S.shard * S.cap + i] = make_int2(tot, rcov);
    S.row_cnt[r] = 0;
  }
}

}  // namespace

cudaError_t launch_shard_top(const ShardArgs& a, uint32_t phase_done, bool apply, bool cond,
                             cudaStream_t s) {
  shard_top_kernel<<<148, 1024, 0, s>>>(a, phase_done, apply ? 1 : 0, cond ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_shard_compact(const ShardArgs& a, bool cond, cudaStream_t s) {
  shard_compact_count_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, cond ? 1 : 0, a.scratch);
  shard_compact_write_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, cond ? 1 : 0, a.scratch);
  return cudaGetLastError();
}

cudaError_t launch_shard_scan(const ShardArgs& a, const int4* req, int nreq, int32_t* cand,
                              int2* meta, cudaStream_t s) {
  if (nreq <= 0) return cudaSuccess;
  // Pieces per request: enough warps to cover the GPU (~16 resident per SM at
  // this kernel's register use) when requests are few, each piece >= one
  // 4 KB warp step, at most kMaxSegs, within the merge buffers.
  const int units = a.thr ? ((a.hi - a.lo) + 31) / 32  // 32-element groups (on the fly)
                          : ((a.hi - a.lo) * a.width + 511) / 512;  // 32-vector units of a slab row
  const int target = 148 * 16;
  int segs = 1;
  if (a.seg_hits && nreq * 2 <= target) {
    segs = std::min(std::min(kMaxSegs, target / nreq), std::max(1, units / 8));
    segs = std::max(1, std::min(segs, kSegWarps / nreq));
  }
  const int blocks = (nreq * segs * 32 + 255) / 256;
  if (a.thr && nreq >= 64) {  // many rows: tile kOtfRows rows over shared point chunks
    const size_t smem = 2 * (size_t)kOtfChunk * (sizeof(double2) + (size_t)a.width) +
                        (size_t)a.thr_n * sizeof(double2);
    const int groups = (nreq + kOtfRows - 1) / kOtfRows;
    const int chunks = (a.hi - a.lo + kOtfChunk - 1) / kOtfChunk;
    // enough blocks for ~4 per SM, pieces of >= 4 chunks, within the merge buffers
    int tsegs = std::max(1, std::min({kMaxSegs, (148 * 4) / groups, chunks / 4, kSegWarps / nreq}));
    if (!a.seg_hits) tsegs = 1;
    // phase 1 (every t(a) == 0 and every target == 0 after init_state): the
    // level-0 test d2 < thr[1] alone, no t stage
    with_width(a.width, [&](auto tag) {
      auto fn = a.first_phase ? shard_scan_otf_tiled_kernel<decltype(tag), true>
                              : shard_scan_otf_tiled_kernel<decltype(tag), false>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      fn<<<groups * tsegs, kOtfRows * 32, smem, s>>>(a, req, nreq, tsegs, cand, meta);
      return 0;
    });
    return cudaGetLastError();
  }
  if (a.thr) {
    const size_t smem = (size_t)a.thr_n * sizeof(double);
    with_width(a.width, [&](auto tag) {
      auto fn = shard_scan_otf_kernel<decltype(tag)>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      fn<<<blocks, 256, smem, s>>>(a, req, nreq, segs, cand, meta);
      return 0;
    });
    return cudaGetLastError();
  }
  with_width(a.width, [&](auto tag) {
    if (a.first_phase)
      shard_scan_kernel<decltype(tag), true><<<blocks, 256, 0, s>>>(a, req, nreq, segs, cand, meta);
    else
      shard_scan_kernel<decltype(tag), false><<<blocks, 256, 0, s>>>(a, req, nreq, segs, cand, meta);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_shard_da(const ShardArgs& a, uint32_t phase, const int32_t* cand,
                            const int2* meta, int nchains, const int4* resume_list,
                            cudaStream_t s) {
  if (nchains <= 0) return cudaSuccess;
  const int blocks = (nchains * 32 + 255) / 256;
  shard_da_kernel<<<blocks, 256, 0, s>>>(a, phase, cand, meta, nchains, resume_list);
  return cudaGetLastError();
}

}  // namespace otprg
