// shard_kernels.cu — the A-row-sharded phase step for several GPUs
// (SURVEY §8(e)).  Shard g owns the demand range [lo_g, hi_g) of every kT
// row; the matching, duals and holders are replicated on every rank and every
// rank runs the same deterministic deferred acceptance, so all ranks hold the
// identical state after each phase and only candidate lists cross NVLink.
//
// Every kernel reads its round parameters (mode, request count, phase, park
// buffer) from the control block, so the same launches run host-driven (one
// host sync per round, torch.distributed exchange: sharded.py) or as the body
// of a CUDA-graph WHILE loop that never returns to the host (resident mode,
// otprg_shard_solve_resident: the exchange is a peer-memory push + flags).
// Per round:
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
#include <cstdlib>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

#ifndef OTPRG_SHARD_UNROLL
#define OTPRG_SHARD_UNROLL 12  // A/B (scripts/ab_shard_unroll.sh): 4 / 8 / 12 / 16 / 24 -> 13.6 / 13.5 / 12.1 / 15.8 / 18.3 ms
#endif

constexpr int kOtfTiledMin = 64;  // requests from which the tiled on-the-fly kernel runs

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

// Round parameters, read by every kernel at its start (written by the ctl
// kernel of the previous round; ld.cg: never from a stale L1 line).
struct Round {
  int mode, nreq;
  uint32_t phase;     // phases completed (the running phase is phase + 1)
  const int4* req;    // mode 1: the parked chains (list index, b, restart)
  int4* park_out;     // chains parked by this round's DA
  bool stop;          // finished or failed: nothing to do
};
__device__ __forceinline__ Round round_of(const ShardArgs& S) {
  const Ctl* c = S.ctl;
  Round r;
  // (sh_live, not done: done is set by the top kernel inside a round)
  r.stop = __ldcg(&c->sh_live) == 0 || __ldcg(&c->status) != 0;
  r.mode = __ldcg(&c->sh_mode);
  r.nreq = r.stop ? 0 : __ldcg(&c->sh_nreq);
  r.phase = __ldcg(&c->phase);
  const int pc = __ldcg(&c->sh_park_cur);
  r.req = r.mode ? S.park[pc] : nullptr;
  r.park_out = S.park[pc ^ 1];
  return r;
}

// Pieces per request of the slab / per-row on-the-fly scans: enough warps to
// cover the GPU (~16 resident per SM) when requests are few, each piece >=
// one 4 KB warp step, at most kMaxSegs, within the merge buffers.
__device__ __forceinline__ int scan_segs(const ShardArgs& S, int nreq) {
  const int units = (S.thr || S.l1x) ? ((S.hi - S.lo) + 31) / 32      // 32-element groups (on the fly)
                          : ((S.hi - S.lo) * S.width + 511) / 512;    // 32-vector units of a slab row
  const int target = 148 * 16;
  int segs = 1;
  if (S.seg_hits && nreq > 0 && nreq * 2 <= target) {
    segs = min(min(kMaxSegs, target / nreq), max(1, units / 8));
    segs = max(1, min(segs, kSegWarps / nreq));
  }
  return segs;
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
template <typename T, bool kP1, bool kSmemT>
__device__ __forceinline__ void scan_slab_item(const ShardArgs& S, const int4* __restrict__ req, int segs,
                                               int w, int32_t* __restrict__ cand, int2* __restrict__ meta,
                                               const uint4* __restrict__ s_t) {
  using SD = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  constexpr int kU = OTPRG_SHARD_UNROLL;  // 16-byte loads in flight per lane (12: 6 KB per warp step)
  const int lane = threadIdx.x & 31;
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
    const uint4* tv = kSmemT ? s_t : reinterpret_cast<const uint4*>(static_cast<const T*>(S.t) + lo);
    const int nv = (width_local + kEpv - 1) / kEpv;
    // this warp's piece, in 32-vector units
    const int u0 = (lstart / kEpv) >> 5, units = (nv + 31) >> 5;
    const int per = (units - u0 + segs - 1) / segs;
    const int vb = (u0 + sg * per) * 32, ve = min(nv, (u0 + (sg + 1) * per) * 32);
    bool full = false;
    for (int v = vb; v < ve && !full; v += 32 * kU) {
      // t from shared memory (kSmemT: read at use) or preloaded with the kT loads
      uint4 kr[kU], tr[(kP1 || kSmemT) ? 1 : kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int vi = v + j * 32 + lane;
        if (vi < ve) {
          kr[j] = __ldg(rv + vi);
          if constexpr (!kP1 && !kSmemT) tr[j] = __ldcg(tv + vi);
        } else {
          kr[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
          if constexpr (!kP1 && !kSmemT) tr[j] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        if (full) break;
        const int vi = v + j * 32 + lane;
        const int e0 = vi * kEpv;  // local element index
        uint4 tj = make_uint4(0u, 0u, 0u, 0u);  // phase 1: t == 0 everywhere (init_state), no t traffic
        if constexpr (!kP1) {
          if constexpr (kSmemT) tj = vi < ve ? tv[vi] : make_uint4(0u, 0u, 0u, 0u);
          else tj = tr[j];
        }
        const uint32_t kw[4] = {kr[j].x, kr[j].y, kr[j].z, kr[j].w};
        const uint32_t tw[4] = {tj.x, tj.y, tj.z, tj.w};
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

// kSmemT: the slab's t staged in shared memory once per launch (the kernel is
// grid-stride: a block serves many rows), so every in-flight load slot of a
// lane carries kT bytes (round 2: the global-t form spent half of them on t).
template <typename T, bool kSmemT>
__global__ void __launch_bounds__(256) shard_scan_kernel(ShardArgs S, int32_t* __restrict__ cand,
                                                         int2* __restrict__ meta) {
  extern __shared__ __align__(16) uint4 s_tslab[];
  const Round rd = round_of(S);
  if (rd.stop) return;
  if (kSmemT && rd.phase != 0) {
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const T*>(S.t) + S.lo);
    const int nv = ((S.hi - S.lo) * (int)sizeof(T) + 15) / 16;
    for (int q = threadIdx.x; q < nv; q += blockDim.x) s_tslab[q] = __ldcg(src + q);
    __syncthreads();
  }
  const int segs = scan_segs(S, rd.nreq);
  const int work = rd.nreq * segs;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < work; w += nwarps) {
    if (rd.phase == 0)  // phase 1: t == 0 everywhere (init_state), no t traffic
      scan_slab_item<T, true, kSmemT>(S, rd.req, segs, w, cand, meta, s_tslab);
    else
      scan_slab_item<T, false, kSmemT>(S, rd.req, segs, w, cand, meta, s_tslab);
  }
}

// Top of a phase: apply M' of the phase the DA just completed (replicated;
// apply_phase, assignment.cpp:210-235), termination / phase cap (:324-334,
// :356-358), counters of the next phase.  first: the top before phase 1
// (nothing to apply).  Skipped while chains are parked (the phase goes on).
// Reads only what earlier kernels wrote (ctl->phase is advanced by the ctl
// kernel), so its blocks never race with its own thread 0.
__device__ __forceinline__ bool top_runs(const Ctl* ctl, int first) {
  if (__ldcg(&ctl->status)) return false;
  return first || (__ldcg(&ctl->work[1]) == 0 && __ldcg(&ctl->sh_live) != 0);
}

__device__ __forceinline__ void top_body(const ShardArgs& S, int first, uint32_t phase_now) {
  Ctl* ctl = S.ctl;
  const uint32_t phase_done = first ? 0u : phase_now + 1u;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gthreads = gridDim.x * blockDim.x;
  const int par = phase_done & 1;
  if (!first) {
    const int2* mp_prev = S.mps + (size_t)par * S.ib;
    const int m = __ldcg(&ctl->mp_cnt[par]);
    for (int q = gtid; q < m; q += gthreads) {
      const int2 e = __ldcg(mp_prev + q);
      const int a = e.x, old_b = e.y;
      const int b = (int)(uint32_t)__ldcg(S.holder + a);
      if (old_b >= 0) S.match_b[old_b] = -1;
      S.match_a[a] = b;
      S.match_b[b] = a;
      const uint32_t nt = t_get(S, a) + 1u;
      if (nt > ctl->tmax) report(ctl, 12, (int)phase_done, a, (int)nt);
      t_set(S, a, nt);
    }
  }
  const int n = __ldcg(&ctl->cnt[par]);
  if (gtid == 0) {
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
      ctl->exh[nx] = 0;
    }
  }
}

__global__ void __launch_bounds__(1024) shard_top_kernel(ShardArgs S, int first) {
  if (!top_runs(S.ctl, first)) return;
  top_body(S, first, __ldcg(&S.ctl->phase));
}

// The free list of the coming phase, ascending b (identical on every rank,
// so list indices name the same b everywhere), and its inverse.  Two passes
// over kCompactBlocks contiguous ranges: per-range counts, then ordered writes
// at the range's offset (block-wide scans per 1024-entry tile).
constexpr int kCompactBlocks = 148;

__device__ __forceinline__ bool compact_skip(const Ctl* c) {
  return __ldcg(&c->done) || __ldcg(&c->status) || __ldcg(&c->work[1]) != 0;
}

__device__ __forceinline__ void compact_count_body(const ShardArgs& S, int* counts) {
  const int n_b = S.ctl->n_b;
  const int chunk = (n_b + gridDim.x - 1) / gridDim.x;
  const int lo = min(n_b, (int)blockIdx.x * chunk), hi = min(n_b, lo + chunk);
  int c = 0;
  for (int q = lo + threadIdx.x; q < hi; q += blockDim.x) c += (__ldcg(S.match_b + q) == -1);
  __shared__ int s_sum;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_sum, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_sum;
}

__global__ void __launch_bounds__(1024) shard_compact_count_kernel(ShardArgs S, int* counts) {
  if (compact_skip(S.ctl)) return;
  compact_count_body(S, counts);
}

__device__ __forceinline__ void compact_write_body(const ShardArgs& S, const int* counts) {
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int n_b = S.ctl->n_b;
  const int chunk = (n_b + gridDim.x - 1) / gridDim.x;
  const int lo = min(n_b, (int)blockIdx.x * chunk), hi = min(n_b, lo + chunk);
  if (threadIdx.x == 0) {
    int off = 0;
    for (int g = 0; g < (int)blockIdx.x; ++g) off += __ldcg(counts + g);
    s_base = off;
  }
  __syncthreads();
  int32_t* out = const_cast<int32_t*>(S.list_in);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int t0 = lo; t0 < hi; t0 += blockDim.x) {  // one tile: block-wide ordered scan of the flags
    const int q = t0 + threadIdx.x;
    const bool f = q < hi && __ldcg(S.match_b + q) == -1;
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

__global__ void __launch_bounds__(1024) shard_compact_write_kernel(ShardArgs S, const int* counts) {
  if (compact_skip(S.ctl)) return;
  compact_write_body(S, counts);
}

// Round bookkeeping (one thread), after the DA (and the top when the phase
// completed): parked chains -> a refill round over them; else the phase is
// complete -> the next phase's first round over its free list.  Sets the
// resident loop's WHILE condition (continue while not finished and no error).
// parked: the DA's parked-chain count (read by the caller before any reset).
__device__ __forceinline__ void ctl_body(const ShardArgs& S, int first, int parked, cudaGraphConditionalHandle cond,
                                        int use_cond) {
  Ctl* c = S.ctl;
  if (!first && !c->sh_live) {  // a loop entered after the solve had finished: nothing ran
    if (use_cond) cudaGraphSetConditional(cond, 0u);
    return;
  }
  if (parked > 0) {
    c->sh_mode = 1;
    c->sh_nreq = parked;
    c->sh_rounds += 1;
  } else {
    if (!first) c->phase += 1;  // the DA's phase is complete (its top ran)
    c->applied = c->phase;
    c->sh_mode = 0;
    c->sh_nreq = c->done ? 0 : c->cnt[c->phase & 1];
  }
  if (!first) {
    c->sh_park_cur ^= 1;
    c->sh_epoch += 1;
  }
  c->work[1] = 0;
  const int go = !c->done && !c->status;
  c->sh_live = go;
  if (use_cond) cudaGraphSetConditional(cond, go ? 1u : 0u);
}

__global__ void shard_ctl_kernel(ShardArgs S, int first, cudaGraphConditionalHandle cond, int use_cond) {
  ctl_body(S, first, first ? 0 : S.ctl->work[1], cond, use_cond);
}

// Everything after a round's DA in ONE cooperative launch (one block per SM,
// co-resident): the top when the phase is complete, the compaction's count
// and write passes, and the round bookkeeping, separated by two grid
// barriers (the monotone arrival counter of device_common.cuh; its base is
// carried across launches in ctl->bar_base).  Every value a later part of
// the kernel changes (work[1], sh_live, phase) is read before the first
// barrier.
__global__ void __launch_bounds__(1024) shard_round_end_kernel(ShardArgs S, int first,
                                                               cudaGraphConditionalHandle cond, int use_cond) {
  Ctl* c = S.ctl;
  unsigned target = ld_cg(reinterpret_cast<const unsigned*>(&c->bar_base));
  const bool runs = top_runs(c, first);
  const int parked = first ? 0 : __ldcg(&c->work[1]);
  const uint32_t phase_now = __ldcg(&c->phase);
  if (runs) top_body(S, first, phase_now);
  target += gridDim.x;
  grid_barrier(c, target);
  const bool compact = runs && !__ldcg(&c->done) && !__ldcg(&c->status);
  if (compact) compact_count_body(S, S.scratch);
  target += gridDim.x;
  grid_barrier(c, target);
  if (compact) compact_write_body(S, S.scratch);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl_body(S, first, parked, cond, use_cond);
    c->bar_base = target;  // every block has passed both barriers
  }
}

// Deferred acceptance over merged candidate lists, one warp per chain
// (grid-stride over the round's chains).  Mode 0: a chain per free b of the
// phase; mode 1: the parked chains resume.
__device__ __forceinline__ void da_chain(const ShardArgs& S, const Round& rd, int w,
                                         const int32_t* __restrict__ cand, const int2* __restrict__ meta) {
  Ctl* ctl = S.ctl;
  const int lane = threadIdx.x & 31;
  const uint32_t phase = rd.phase + 1u;
  const uint32_t cur_tag = ~phase;
  const int par = phase & 1;
  int i, b, start;
  if (rd.req) {
    const int4 r = __ldcg(rd.req + w);
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
      // the slot's candidates are loaded with its meta (one round trip), then
      // cut to the meta's count
      const int cc = lane < K ? __ldcg(cand + ((size_t)g * S.cap + i) * K + lane) : -1;
      const int2 mt = __ldcg(meta + (size_t)g * S.cap + i);
      const int c = lane < mt.x ? cc : -1;
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
        rd.park_out[pos] = make_int4(i, b, restart, 0);
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
      S.mps[(size_t)par * S.ib + pos] = make_int2(a, partner);
    }
    return;
  }
}

__global__ void __launch_bounds__(256) shard_da_kernel(ShardArgs S, const int32_t* __restrict__ cand,
                                                       const int2* __restrict__ meta) {
  const Round rd = round_of(S);
  if (rd.stop) return;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rd.nreq; w += nwarps)
    da_chain(S, rd, w, cand, meta);
}

// Peer exchange of a device group (resident multi-GPU loop): push the local
// shards' slots of this round (nreq rows) into every peer group's exchange
// buffers over NVLink peer memory, then — last block — release this round's
// epoch into every peer's flag array and wait (acquire, system scope) until
// every peer's flag in ours reached it.  Epochs only grow (never reset), so a
// peer that runs ahead can never be missed.  A wait longer than 20 s reports
// status 6 (device) and the loop ends instead of hanging.
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// blk / nblk: this block's index among the blocks pushing for the group.
__device__ __forceinline__ void push_body(const ShardArgs& S, const int32_t* __restrict__ cand,
                                          const int2* __restrict__ meta, const ShardPeers& P, int blk, int nblk) {
  const Round rd = round_of(S);
  if (rd.stop) return;
  const uint32_t epoch = __ldcg(&S.ctl->sh_epoch) + 1u;
  const int nreq = rd.nreq, K = S.K;
  const size_t tid = (size_t)blk * blockDim.x + threadIdx.x, nthr = (size_t)nblk * blockDim.x;
  for (int g = P.shard_lo; g < P.shard_hi; ++g) {
    const size_t c0 = (size_t)g * S.cap * K, m0 = (size_t)g * S.cap;
    const size_t nc = (size_t)nreq * K;
    for (int p = 0; p < P.n; ++p) {
      for (size_t q = tid; q < nc; q += nthr) P.cand[p][c0 + q] = __ldcg(cand + c0 + q);
      for (size_t q = tid; q < (size_t)nreq; q += nthr) P.meta[p][m0 + q] = __ldcg(meta + m0 + q);
    }
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(P.arrive, 1u) == (unsigned)nblk - 1u;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  *P.arrive = 0;  // ready for the next round
  __threadfence_system();
  for (int p = 0; p < P.n; ++p) st_release_sys(P.flag[p] + P.my_group, epoch);
  const unsigned long long t0 = globaltimer();
  for (int q = 0; q < P.n_groups; ++q) {
    if (q == P.my_group) continue;
    while ((int)(ld_acquire_sys(P.my_flags + q) - epoch) < 0) {
      if (globaltimer() - t0 > 20000000000ull) {
        report(S.ctl, 6, -2, q, (int)epoch);
        return;
      }
    }
  }
}

__global__ void __launch_bounds__(256) shard_push_kernel(ShardArgs S, const int32_t* __restrict__ cand,
                                                         const int2* __restrict__ meta, ShardPeers P) {
  push_body(S, cand, meta, P, blockIdx.x, gridDim.x);
}

// Self-test of the exchange protocol on ONE device: every group's push runs
// as a slice of one cooperative grid (all blocks co-resident), so the groups'
// flag waits are satisfied by blocks that are guaranteed to run — the
// emulation the multi-GPU push needs on a single GPU.
__global__ void __launch_bounds__(256) shard_push_emulate_kernel(const ShardArgs* __restrict__ S,
                                                                 const int32_t* const* __restrict__ cand,
                                                                 const int2* const* __restrict__ meta,
                                                                 const ShardPeers* __restrict__ P, int nblk) {
  const int g = blockIdx.x / nblk;
  push_body(S[g], cand[g], meta[g], P[g], blockIdx.x - g * nblk, nblk);
}

// On-the-fly variant (OTPRG_FLAG_ON_THE_FLY): no kT slab.  Each lane
// takes one demand point per 32-element group, forms d2 = dx*dx + dy*dy in
// IEEE round-to-nearest (the reference's bits, instances.cpp:70-75) and tests
// admissibility k(a,b) + t(a) == target as thr[m] <= d2 < thr[m+1] with
// m = target - t(a), against the exact threshold table staged in shared
// memory: no sqrt, no division, 16 B of point per element instead of w B of kT.
// Outputs, pieces and the merge as shard_scan_kernel.
template <typename T>
__device__ __forceinline__ void scan_otf_item(const ShardArgs& S, const double* __restrict__ s_thr,
                                              const int4* __restrict__ req, int segs, int w,
                                              int32_t* __restrict__ cand, int2* __restrict__ meta) {
  constexpr int kG = 8;  // 32-element groups per warp step
  const int lane = threadIdx.x & 31;
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


// On-the-fly L1 image costs (load_mnist_pair's cost, instances.cpp:134-141;
// north star (1): costs from d-dim vectors when the matrix does not fit).
// A warp per (request, piece): the supply image's normalised pixels sit in
// the warp's shared-memory slice, each lane sums |x_a[p] - y_b[p]| over
// ascending p for its demand vertex (pixels transposed [p][a]: a warp reads 32
// consecutive a per p), halves it and rounds it exactly (scaled_floor), the
// reference's bits; admissible iff k + t(a) == Y(b) - 1.  FP64-bound (2 dim
// operations per entry), which is why the materialised matrix is preferred
// whenever it fits.  Outputs, pieces and the merge as the other scans.
template <typename T>
__device__ __forceinline__ void scan_l1_item(const ShardArgs& S, double* __restrict__ s_y, const int4* __restrict__ req,
                                             int segs, int w, int32_t* __restrict__ cand, int2* __restrict__ meta) {
  const int lane = threadIdx.x & 31;
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
  const int lo = S.lo, hi = S.hi, K = S.K, width_local = hi - lo, dim = S.dim;
  const size_t na_full = (size_t)S.na_full;
  int32_t* o = segs == 1 ? cand + ((size_t)S.shard * S.cap + i) * K : S.seg_hits + (size_t)w * K;
  int cnt = 0, cov = hi;
  const int lstart = max(start, lo) - lo;
  __syncwarp();
  for (int p = lane; p < dim; p += 32) s_y[p] = S.l1y[(size_t)b * dim + p];
  __syncwarp();
  if (start < hi) {
    const T* tl = static_cast<const T*>(S.t) + lo;
    const int groups = (width_local + 31) >> 5, g0 = lstart >> 5;
    const int per = (groups - g0 + segs - 1) / segs;
    const int gb = g0 + sg * per, ge = min(groups, g0 + (sg + 1) * per);
    for (int g = gb; g < ge; ++g) {
      const int e = g * 32 + lane;
      bool hit = false;
      if (e < width_local && e >= lstart) {
        const double* x = S.l1x + lo + e;
        double acc = 0.0;
        // ascending p over the union of the group's and b's pixel supports
        // (a pixel zero in both adds +0: the sum's bits are unchanged)
        const int nw = (dim + 31) >> 5;
        const uint32_t* gm = S.l1_gmask + (size_t)g * nw;
        const uint32_t* bm = S.l1_bmask + (size_t)b * nw;
        for (int wd = 0; wd < nw; ++wd) {
          uint32_t m = __ldg(gm + wd) | __ldg(bm + wd);
          while (m) {
            const int p = (wd << 5) + __ffs(m) - 1;
            m &= m - 1;
            acc = __dadd_rn(acc, fabs(__dsub_rn(__ldg(x + (size_t)p * na_full), s_y[p])));
          }
        }
        const long long k = scaled_floor_dev(__ddiv_rn(acc, 2.0), S.eps);
        hit = k + (long long)__ldcg(tl + e) == target;
      }
      const unsigned bal = __ballot_sync(kFull, hit);
      if (!bal) continue;
      const int idx = cnt + __popc(bal & ((1u << lane) - 1u));
      if (hit && idx < K) o[idx] = lo + e;
      const int c = __popc(bal);
      if (cnt + c >= K) {
        unsigned bm = bal;
        for (int t2 = 1; t2 < K - cnt; ++t2) bm &= bm - 1;
        cov = lo + g * 32 + __ffs(bm);
        cnt = K;
        break;
      }
      cnt += c;
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

template <typename T>
__global__ void __launch_bounds__(256) shard_scan_l1_kernel(ShardArgs S, int32_t* __restrict__ cand,
                                                            int2* __restrict__ meta) {
  const Round rd = round_of(S);
  if (rd.stop) return;
  extern __shared__ double s_l1y[];  // [warps per block][dim]
  double* s_y = s_l1y + (size_t)(threadIdx.x >> 5) * S.dim;
  const int segs = scan_segs(S, rd.nreq);
  const int work = rd.nreq * segs;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < work; w += nwarps)
    scan_l1_item<T>(S, s_y, rd.req, segs, w, cand, meta);
}

// Few requests (or no room for the tiled kernel): a warp per (request, piece).
template <typename T>
__global__ void __launch_bounds__(256) shard_scan_otf_kernel(ShardArgs S, int32_t* __restrict__ cand,
                                                             int2* __restrict__ meta) {
  const Round rd = round_of(S);
  if (rd.stop || (S.otf_tiled && rd.nreq >= kOtfTiledMin)) return;
  extern __shared__ double s_thr[];
  for (int j = threadIdx.x; j < S.thr_n; j += blockDim.x) s_thr[j] = S.thr[j];
  __syncthreads();
  const int segs = scan_segs(S, rd.nreq);
  const int work = rd.nreq * segs;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < work; w += nwarps)
    scan_otf_item<T>(S, s_thr, rd.req, segs, w, cand, meta);
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

struct OtfTileSmem {
  unsigned long long* bar;  // [2] stage barriers
  int* lo_start;
  int* act;                 // [3]
  const double2* pair;      // (thr[m], thr[m+1])
};

// One work item of the tiled on-the-fly scan: row group grp's piece sg.
// `par` carries the stage barriers' phase bits across items.
template <typename T, bool kP1>
__device__ __forceinline__ void otf_tile_item(const ShardArgs& S, unsigned char* s_dyn, const OtfTileSmem& sm,
                                              const int4* __restrict__ req, int nreq, int segs, int item,
                                              unsigned& par, int32_t* __restrict__ cand,
                                              int2* __restrict__ meta) {
  // stage st: points [kOtfChunk] double2 then t [kOtfChunk] T; the pair table after both stages
  constexpr size_t kStage = (size_t)kOtfChunk * (sizeof(double2) + sizeof(T));
  const double2* s_pair = sm.pair;
  unsigned long long* bar = sm.bar;
  int& s_lo_start = *sm.lo_start;
  int* s_act = sm.act;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = item / segs, sg = item - grp * segs;
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
  }
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
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();  // the stages were read (generic proxy) by the previous item
    for (int k = 0; k < min(2, nchunk); ++k) issue(k);
  }
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
  if (k < nchunk) {
    if (threadIdx.x == 0) mbar_wait(&bar[k & 1], (par >> (k & 1)) & 1u);
    par ^= 1u << (k & 1);
  }
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

template <typename T>
__global__ void __launch_bounds__(kOtfRows * 32) shard_scan_otf_tiled_kernel(ShardArgs S, int32_t* __restrict__ cand,
                                                                            int2* __restrict__ meta) {
  const Round rd = round_of(S);
  if (rd.stop || !S.otf_tiled || rd.nreq < kOtfTiledMin) return;
  extern __shared__ __align__(128) unsigned char s_dyn[];
  constexpr size_t kStage = (size_t)kOtfChunk * (sizeof(double2) + sizeof(T));
  double2* s_pair = reinterpret_cast<double2*>(s_dyn + 2 * kStage);
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ int s_lo_start, s_act[3];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = threadIdx.x; j + 1 < S.thr_n; j += blockDim.x) s_pair[j] = make_double2(S.thr[j], S.thr[j + 1]);
  __syncthreads();
  const OtfTileSmem sm{bar, &s_lo_start, s_act, s_pair};
  const int nreq = rd.nreq;
  const int groups = (nreq + kOtfRows - 1) / kOtfRows;
  const int chunks = (S.hi - S.lo + kOtfChunk - 1) / kOtfChunk;
  // pieces per row group: the grid's blocks over the groups, pieces of >= 4
  // chunks, within the merge buffers
  int segs = max(1, min(min(kMaxSegs, (int)gridDim.x / groups), min(chunks / 4, kSegWarps / nreq)));
  if (!S.seg_hits) segs = 1;
  unsigned par = 0;
  for (int item = blockIdx.x; item < groups * segs; item += gridDim.x) {
    // phase 1 (every t(a) == 0 and every target == 0 after init_state): the
    // level-0 test d2 < thr[1] alone, no t stage
    if (rd.phase == 0) otf_tile_item<T, true>(S, s_dyn, sm, rd.req, nreq, segs, item, par, cand, meta);
    else otf_tile_item<T, false>(S, s_dyn, sm, rd.req, nreq, segs, item, par, cand, meta);
    __syncthreads();
  }
}

}  // namespace

namespace {
size_t otf_tiled_smem(int width, int thr_n) {
  return 2 * (size_t)kOtfChunk * (sizeof(double2) + (size_t)width) + (size_t)thr_n * sizeof(double2);
}
// Resident blocks per SM of a kernel at its launch shape (>= 1).
template <typename K>
int blocks_per_sm(K fn, int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess || n < 1) n = 1;
  return n;
}
}  // namespace

// Shared memory for the slab's t in the slab scan (0: too large, t from L2).
// Off by default: A/B on config 4 (G = 1, u8, resident; scripts/probe_k.py):
// 9.2-9.6 ms with t from L2, 9.6-10.3 ms staged — every launch restages the
// slab's t per block (296 blocks x 100 KB from L2 per round) and occupancy
// does not rise (2 blocks per SM either way).  OTPRG_SLAB_TSMEM=1 turns it on.
size_t slab_t_smem(const ShardArgs& a) {
  static const bool on = [] {
    const char* e = std::getenv("OTPRG_SLAB_TSMEM");
    return e && e[0] == '1';
  }();
  const size_t bytes = ((size_t)(a.hi - a.lo) * a.width + 15) / 16 * 16;
  return on && bytes <= 96 * 1024 ? std::max<size_t>(bytes, 16) : 0;
}

static_assert(kOtfChunk % (32 * OTPRG_OTF_GU) == 0, "OTPRG_OTF_CHUNK must be a multiple of 32 * OTPRG_OTF_GU");
static_assert((kOtfChunk * 16) % 16 == 0 && kOtfChunk % 16 == 0, "OTPRG_OTF_CHUNK must keep 16-byte stages");

// Grid of the scan kernels: every SM filled with resident blocks (the
// kernels loop over their work items, whose count is only known on the device).
int shard_scan_grid(const ShardArgs& a, int num_sms) {
  int g = 0;
  with_width(a.width, [&](auto tag) {
    using T = decltype(tag);
    if (a.l1x) {
      const size_t smem = (size_t)8 * a.dim * sizeof(double);
      smem_attr_raise(shard_scan_l1_kernel<T>, smem);
      g = num_sms * blocks_per_sm(shard_scan_l1_kernel<T>, 256, smem);
    } else if (a.thr) {
      const int simple = blocks_per_sm(shard_scan_otf_kernel<T>, 256, (size_t)a.thr_n * sizeof(double));
      g = num_sms * simple;
      if (a.otf_tiled) {
        const size_t smem = otf_tiled_smem(a.width, a.thr_n);
        smem_attr_raise(shard_scan_otf_tiled_kernel<T>, smem);
        g = std::max(g, num_sms * blocks_per_sm(shard_scan_otf_tiled_kernel<T>, kOtfRows * 32, smem));
      }
    } else {
      const size_t st = slab_t_smem(a);
      if (st) {
        smem_attr_raise(shard_scan_kernel<T, true>, st);
        g = num_sms * blocks_per_sm(shard_scan_kernel<T, true>, 256, st);
      } else {
        g = num_sms * blocks_per_sm(shard_scan_kernel<T, false>, 256, 0);
      }
    }
    return 0;
  });
  return g;
}

// Whether the tiled on-the-fly kernel's stages + pair table fit the opt-in
// shared-memory limit (else the per-row kernel serves every request count).
bool shard_otf_tiled_fits(int width, int thr_n, int device) {
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return otf_tiled_smem(width, thr_n) <= (size_t)optin;
}

cudaError_t launch_shard_scan(const ShardArgs& a, int32_t* cand, int2* meta, int grid, cudaStream_t s) {
  with_width(a.width, [&](auto tag) {
    using T = decltype(tag);
    if (a.l1x) {
      const size_t smem = (size_t)8 * a.dim * sizeof(double);
      auto fn = shard_scan_l1_kernel<T>;
      smem_attr_raise(fn, smem);
      fn<<<grid, 256, smem, s>>>(a, cand, meta);
    } else if (a.thr) {
      const size_t smem1 = (size_t)a.thr_n * sizeof(double);
      auto fn1 = shard_scan_otf_kernel<T>;
      smem_attr_raise(fn1, smem1);
      // each of the two exits at once unless the round's request count is its regime
      fn1<<<grid, 256, smem1, s>>>(a, cand, meta);
      if (a.otf_tiled) {
        const size_t smem = otf_tiled_smem(a.width, a.thr_n);
        auto fn = shard_scan_otf_tiled_kernel<T>;
        smem_attr_raise(fn, smem);
        fn<<<grid, kOtfRows * 32, smem, s>>>(a, cand, meta);
      }
    } else {
      const size_t st = slab_t_smem(a);
      if (st) shard_scan_kernel<T, true><<<grid, 256, st, s>>>(a, cand, meta);
      else shard_scan_kernel<T, false><<<grid, 256, 0, s>>>(a, cand, meta);
    }
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_shard_push(const ShardArgs& a, const int32_t* cand, const int2* meta,
                              const ShardPeers& p, cudaStream_t s) {
  shard_push_kernel<<<148, 256, 0, s>>>(a, cand, meta, p);
  return cudaGetLastError();
}

cudaError_t launch_shard_push_emulated(const ShardArgs* a, const int32_t* const* cand, const int2* const* meta,
                                       const ShardPeers* p, int n_groups, int nblk, cudaStream_t s) {
  void* args[] = {(void*)&a, (void*)&cand, (void*)&meta, (void*)&p, (void*)&nblk};
  return cudaLaunchCooperativeKernel((const void*)shard_push_emulate_kernel, dim3(n_groups * nblk), dim3(256),
                                     args, 0, s);
}

cudaError_t launch_shard_da(const ShardArgs& a, const int32_t* cand, const int2* meta, int grid,
                            cudaStream_t s) {
  shard_da_kernel<<<grid, 256, 0, s>>>(a, cand, meta);
  return cudaGetLastError();
}

cudaError_t launch_shard_after_da(const ShardArgs& a, cudaStream_t s) {
  shard_top_kernel<<<148, 1024, 0, s>>>(a, 0);
  shard_compact_count_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, a.scratch);
  shard_compact_write_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, a.scratch);
  return cudaGetLastError();
}

cudaError_t launch_shard_ctl(const ShardArgs& a, cudaGraphConditionalHandle cond, bool use_cond,
                             cudaStream_t s) {
  shard_ctl_kernel<<<1, 1, 0, s>>>(a, 0, cond, use_cond ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_shard_round_end(const ShardArgs& a, cudaGraphConditionalHandle cond, bool use_cond,
                                   cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCompactBlocks);
  cfg.blockDim = dim3(1024);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, shard_round_end_kernel, a, 0, cond, use_cond ? 1 : 0);
}

cudaError_t launch_shard_first_top(const ShardArgs& a, cudaStream_t s) {
  shard_top_kernel<<<148, 1024, 0, s>>>(a, 1);
  shard_compact_count_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, a.scratch);
  shard_compact_write_kernel<<<kCompactBlocks, 1024, 0, s>>>(a, a.scratch);
  shard_ctl_kernel<<<1, 1, 0, s>>>(a, 1, cudaGraphConditionalHandle{}, 0);
  return cudaGetLastError();
}

}  // namespace otprg
