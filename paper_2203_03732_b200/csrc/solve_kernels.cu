// solve_kernels.cu — the device-resident phase loop of the push-relabel
// assignment solver (reference: src/assignment.cpp:316-364), for sm_100a.
//
// One persistent cooperative kernel runs whole phases with no host sync and
// ONE grid barrier per phase.  Phase p (free supply set B'_p, target
// Y(b) - 1 for each free b):
//
//  top    Every block applies M'_{p-1} to its shared-memory copy of
//         t(a) = -Y(a) (Y(a) -= 1 for a matched in M', apply_phase :210-235);
//         all threads together apply M'_{p-1} to the global matching
//         (link, drop the displaced partner) and to global t.  Termination
//         (:330-334: n_i <= floor(eps*m)) and the phase cap (:326,356-358)
//         are tested here, after the apply, so the state is consistent at
//         every exit.
//  P      Proposal chains (collect_workset/scan_plain :107-147,65-75 and the
//         sequential greedy :161-171).  Every warp takes a free b and runs a
//         deferred-acceptance chain: find the first admissible a >= start
//         (k(a,b) + t(a) == Y(b) - 1, i.e. Y(a)+Y(b) == k+1) and propose with
//         one 64-bit atomicMin on holder[a] (key = ~phase << 32 | b: lower b
//         wins, older phases lose).  Rejected -> next admissible a of the same
//         row.  Winning over a same-phase holder b2 -> the warp continues
//         b2's chain after a.  No admissible a left -> b stays free:
//         Y(b) += 1 and b joins the next free list.  The first proposal that
//         takes an a this phase also frees a's previous partner (it joins the
//         next free list) and records (a, partner) for the next phase's top.
//         Deferred acceptance with a common priority (lower b first) reaches
//         the serial-dictatorship matching in any proposal order, which is
//         the reference's sequential greedy M' exactly.
//  barrier
//
// Finding admissible edges.  A warp streams the row kT[b][*] (B-major, 1 or
// 2 bytes per entry) with 128-bit loads against t in shared memory, using
// packed saturating SIMD sums.  Each scan from position 0 also records the
// row's "low set": the ascending positions with k + t <= target + 2 (up to
// kLowCap entries, with k).  Since t(a) only grows and Y(b) only grows, the
// admissible set of b at any later target <= that bound is a subset of the
// low set, so later phases verify a handful of cached entries against the
// current t instead of rescanning the row; a row is rescanned only when the
// bound expires or the cache was truncated.  rowmin[b] (min of k + t at the
// last full scan) skips rows that cannot have admissible edges at all.
#include <climits>
#include <cstdio>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

#ifndef OTPRG_BLOCK
#define OTPRG_BLOCK 512  // 16 warps/SM: 128 registers, no spills (768/1024 spill)
#endif
constexpr int kBlock = OTPRG_BLOCK;
#ifndef OTPRG_TEAMS
#define OTPRG_TEAMS 1
#endif
constexpr bool kTeams = OTPRG_TEAMS != 0;  // multi-warp rows in small phases
#ifndef OTPRG_TEAM_OVERSUB
#define OTPRG_TEAM_OVERSUB 1
#endif
#ifndef OTPRG_TEAM_DEN
#define OTPRG_TEAM_DEN 1
#endif
#ifndef OTPRG_STATIC
#define OTPRG_STATIC 1
#endif
// Static slots (small phases): the chain of input slot i writes output slot i
// and its team keeps the next proposer's prologue in registers (no list read
// at the next top).
constexpr bool kStatic = OTPRG_STATIC != 0;
#ifndef OTPRG_STATIC_HOLES
#define OTPRG_STATIC_HOLES 16  // static slots while holes <= 1/this of the slots (A/B: 2 / 4 / 8 / 16)
#endif
#ifndef OTPRG_BULK
#define OTPRG_BULK 1
#endif
#ifndef OTPRG_TAIL
#define OTPRG_TAIL 1  // small phases (teams of 8 warps) run in a second, specialised launch
#endif
#ifndef OTPRG_TAIL_UNROLL
#define OTPRG_TAIL_UNROLL 5  // 128-bit loads in flight per lane in the tail's row scans (A/B 4/5/6/8: a team step of 8 warps then covers 20 KB, one n = 10k uint16 row)
#endif
#ifndef OTPRG_MID
#define OTPRG_MID 1  // the phases with teams of 4 in their own specialised launch too
#endif
#ifndef OTPRG_MID_UNROLL
#define OTPRG_MID_UNROLL 4  // (A/B 4 / 5 / 6 / 8: 2.953 / 2.958 / 2.967 / 2.970 ms)
#endif
#ifndef OTPRG_TAIL_CONST
#define OTPRG_TAIL_CONST 1  // the tail launch with a compile-time team size
#endif
constexpr bool kBulk = OTPRG_BULK != 0;  // streaming list build in large phases
constexpr int kUnroll = 4;       // 128-bit loads in flight per lane (global t)
#ifndef OTPRG_UNROLL_SMEM
#define OTPRG_UNROLL_SMEM 4  // A/B (scripts/ab_unroll.sh): 2 / 4 / 6 / 8 / 16 -> 3.44 / 3.34 / 3.46 / 3.72 / 5.21 ms
#endif
constexpr int kUnrollSmem = OTPRG_UNROLL_SMEM;  // (t in shared memory)

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) { return __ldg(p); }

template <bool kSmem>
__device__ __forceinline__ uint4 load_t(const uint4* p) {
  if constexpr (kSmem) return *p;
  else return __ldcg(p);
}

// Low-set construction state of the current scan (uniform across the warp).
struct LowBuild {
  bool on = false;
  int cnt = 0;                        // entries stored so far
  int full_pos = -1;                  // position of the kLowCap-th entry once full
  uint32_t up_rep = 0;                // packed upper level
  unsigned long long* ent = nullptr;  // &lent[b * kLowCap]
};

template <typename S>
__device__ __forceinline__ uint32_t pick_word(int i, uint32_t w0, uint32_t w1, uint32_t w2,
                                              uint32_t w3) {
  const int q = i / S::kEpw;
  return q < 2 ? (q == 0 ? w0 : w1) : (q == 2 ? w2 : w3);
}

// A team of `size` consecutive warps of one block that works on one proposer
// chain together (used when a phase has few proposers, so each row scan is
// split across warps).  size == 1 is the plain warp-per-proposer mode.
struct Team {
  int size;                  // 1, 2, 4 or 8 warps
  int rank;                  // warp index within the team
  unsigned bar;              // named barrier id (1..15) when size > 1
  unsigned long long* slot;  // shared-memory broadcast area (>= 9 words)
};

__device__ __forceinline__ void team_sync(const Team& tm) {
  if (tm.size > 1) asm volatile("bar.sync %0, %1;" ::"r"(tm.bar), "r"(tm.size * 32) : "memory");
}

// value of the team leader (rank 0, lane 0), everywhere in the team
__device__ __forceinline__ unsigned long long team_bcast(const Team& tm, unsigned long long v,
                                                         int lane) {
  if (tm.size == 1) return __shfl_sync(kFull, v, 0);
  if (tm.rank == 0 && lane == 0) tm.slot[0] = v;
  team_sync(tm);
  const unsigned long long r = tm.slot[0];
  team_sync(tm);
  return r;
}

// min over the team of a warp-uniform value
__device__ __forceinline__ int team_min(const Team& tm, int v, int lane) {
  if (tm.size == 1) return v;
  if (lane == 0) tm.slot[1 + tm.rank] = (unsigned long long)(unsigned)v;
  team_sync(tm);
  int m = INT_MAX;
  for (int r = 0; r < tm.size; ++r) m = min(m, (int)(unsigned)tm.slot[1 + r]);
  team_sync(tm);
  return m;
}

// First admissible a >= start in one kT row, or -1.  Each warp streams its
// part of the row in 32 lanes x 16 B x kU chunks (coalesced 128-bit loads,
// kU in flight per lane); a team of warps covers consecutive chunks and
// agrees on the first hit per step.  track_min folds min_a (k + t) into mnw;
// lb (warp mode only) appends the low-set entries at positions <= the hit.
template <typename T, bool kSmem, int kUS = kUnrollSmem>
__device__ __forceinline__ int warp_scan(const T* __restrict__ row, const T* tvec, int lda,
                                         int start, uint32_t target, bool track_min,
                                         uint32_t& mnw, LowBuild& lb, int lane, const Team& tm,
                                         unsigned long long& bytes, bool full_row = false) {
  using S = Simd<T>;
  constexpr int kEpv = 16 / sizeof(T);
  const uint32_t tg = S::rep(target);
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  const uint4* tv = reinterpret_cast<const uint4*>(tvec);
  const int nv = lda / kEpv;  // multiple of 32
  constexpr int kU = kSmem ? kUS : kUnroll;
  const int tstride = tm.size * 32 * kU;
  for (int vt = (start / kEpv) & ~31; vt < nv; vt += tstride) {
    const int v = vt + tm.rank * 32 * kU;  // this warp's chunk of the team step
    int first = INT_MAX;
    // kT loads for the whole chunk are issued first (kU in flight per lane);
    // t comes from shared memory at use (or is preloaded when it is global).
    uint4 kr[kU], tr[kSmem ? 1 : kU];
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int vi = v + j * 32 + lane;
      if (vi < nv) {
        kr[j] = ldg_nc(rv + vi);
        if constexpr (!kSmem) tr[j] = load_t<false>(tv + vi);
      } else {
        kr[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
        if constexpr (!kSmem) tr[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    if (lane == 0 && v < nv) bytes += 16ull * (unsigned long long)min(nv - v, 32 * kU);
#pragma unroll
    for (int j = 0; j < kU; ++j) {
      const int vi = v + j * 32 + lane;
      const int e0 = vi * kEpv;
      uint4 tj;
      if constexpr (kSmem) tj = vi < nv ? tv[vi] : make_uint4(0u, 0u, 0u, 0u);
      else tj = tr[j];
      const uint32_t k0 = kr[j].x, k1 = kr[j].y, k2 = kr[j].z, k3 = kr[j].w;
      const uint32_t s0 = S::add(k0, tj.x), s1 = S::add(k1, tj.y);
      const uint32_t s2 = S::add(k2, tj.z), s3 = S::add(k3, tj.w);
      if (track_min) mnw = S::mn(S::mn(mnw, S::mn(s0, s1)), S::mn(s2, s3));
      {  // fast path: nothing admissible (nor low) in this sub-chunk for the whole warp
        uint32_t any = S::eq(s0, tg) | S::eq(s1, tg) | S::eq(s2, tg) | S::eq(s3, tg);
        if (lb.on)
          any |= S::le(s0, lb.up_rep) | S::le(s1, lb.up_rep) | S::le(s2, lb.up_rep) |
                 S::le(s3, lb.up_rep);
        if (!__any_sync(kFull, any != 0)) continue;
      }
      uint32_t eqb = S::bits(S::eq(s0, tg)) | (S::bits(S::eq(s1, tg)) << S::kEpw) |
                     (S::bits(S::eq(s2, tg)) << (2 * S::kEpw)) |
                     (S::bits(S::eq(s3, tg)) << (3 * S::kEpw));
      uint32_t keep = ~0u;
      if (e0 < start) {
        const int drop = start - e0;
        keep = drop >= kEpv ? 0u : (~0u << drop);
        eqb &= keep;
      }
      const unsigned hb = __ballot_sync(kFull, eqb != 0);
      int hit = INT_MAX;
      if (hb) hit = __shfl_sync(kFull, e0 + __ffs(eqb) - 1, __ffs(hb) - 1);
      if (lb.on) {
        uint32_t leb = (S::bits(S::le(s0, lb.up_rep)) | (S::bits(S::le(s1, lb.up_rep)) << S::kEpw) |
                        (S::bits(S::le(s2, lb.up_rep)) << (2 * S::kEpw)) |
                        (S::bits(S::le(s3, lb.up_rep)) << (3 * S::kEpw))) & keep;
        if (hit != INT_MAX && !full_row) {  // entries up to and including the hit only
          const int lim = hit - e0;
          leb = lim < 0 ? 0u : (lim >= kEpv - 1 ? leb : (leb & ((2u << lim) - 1u)));
        }
        if (__ballot_sync(kFull, leb != 0)) {
          const int c = __popc(leb);
          int inc = c;  // inclusive warp scan of the per-lane counts
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
          }
          const int tot = __shfl_sync(kFull, inc, 31);
          int idx = lb.cnt + inc - c;
          const int first_idx = idx;
          uint32_t bm = leb;
          int fp = -1;
          while (bm) {
            const int i = __ffs(bm) - 1;
            bm &= bm - 1;
            if (idx < kLowCap) {
              const uint32_t kv = S::elem(pick_word<S>(i, k0, k1, k2, k3), i % S::kEpw);
              lb.ent[idx] = ((unsigned long long)kv << 32) | (uint32_t)(e0 + i);
              if (idx == kLowCap - 1) fp = e0 + i;
            }
            ++idx;
          }
          if (lb.cnt + tot >= kLowCap) {  // full: coverage ends at the last stored entry
            const unsigned src = __ballot_sync(kFull, first_idx <= kLowCap - 1 &&
                                                          kLowCap - 1 < first_idx + c);
            lb.full_pos = __shfl_sync(kFull, fp, __ffs(src) - 1);
            lb.cnt = kLowCap;
            lb.on = false;
          } else {
            lb.cnt += tot;
          }
        }
      }
      if (hit != INT_MAX && !full_row) {
        first = hit;
        break;
      }
    }
    const int h = team_min(tm, first, lane);
    if (h != INT_MAX) return h;
  }
  return -1;
}

// Per-phase list pointers (selected once so no parameter array is indexed
// dynamically, which would spill the kernel parameters to local memory).
struct PhasePtrs {
  int32_t* list_out;  // free b's of the next phase
  int2* mp_out;       // (a, previous partner) first held this phase
  int* cnt_out;       // free b's of the next phase (count only: red.add)
  int* mp_cnt_out;    // first takes (count only)
  int* exh_out;       // exhausted b's (count only)
  int* slot_out;      // output slot reservations: one per chain
};

// A proposer's chain prologue (Y(b), low-set meta/entries, row min), loaded
// at the top of the phase together with the phase counters so the first
// chain of every warp starts without further dependent loads -- or, after a
// static-slot phase, carried in registers from the chain that produced it.
struct Prefetch {
  bool ok;
  int i, b;
  uint32_t yb, rowmin;
  int4 meta;
  unsigned long long ent;
};

template <typename T, bool kSmem, bool kTail, int kMid = 0>
__device__ __forceinline__ void run_chain(int b, const SolveArgs& A, const PhasePtrs& P,
                                          const T* tp, int lda, uint32_t phase, uint32_t tmax,
                                          int lane, unsigned long long& bytes,
                                          unsigned long long& steps, unsigned long long& walks,
                                          unsigned* s_stat, unsigned long long* acc,
                                          const Team& tm, const Prefetch& pf, bool use_pf,
                                          int in_slot, Prefetch& nx) {
  const bool lead = lane == 0 && tm.rank == 0;  // performs the chain's global side effects
#define OTPRG_STAT(k) \
  if (lead) atomicAdd(&s_stat[k], 1u)
  OTPRG_STAT(0);
  // Every chain ends in exactly one event (b exhausted, or a first take of
  // some a), written to its own output slot: the slot is reserved now, so
  // the reservation's round trip overlaps the chain instead of ending it.
  // Static slots: output slot = input slot (in_slot >= 0), the next
  // proposer's prologue goes to nx (nx.ok = false: reload it at the top).
  int slot = in_slot;
  if (lead && in_slot < 0) slot = atomicAdd(P.slot_out, 1);
  using S = Simd<T>;
  Ctl* ctl = A.ctl;
  const T* kT = static_cast<const T*>(A.kT);
  T* rowmin = static_cast<T*>(A.rowmin);
  const uint32_t cur_tag = ~phase;
  const uint32_t prev_tag = ~(phase - 1);
  unsigned long long* H = (phase & 1) ? A.holder[1] : A.holder[0];             // this phase
  const unsigned long long* Hprev = (phase & 1) ? A.holder[0] : A.holder[1];   // phase - 1

  uint32_t yb;
  int4 meta;  // low-set cache of b: (upto, cov, cnt, -)
  unsigned long long ent = 0;
  uint32_t rmin;
  if (use_pf) {
    yb = pf.yb;
    meta = pf.meta;
    ent = pf.ent;
    rmin = pf.rowmin;
  } else {
    yb = (uint32_t)__ldcg(A.yb + b);
    meta = __ldcg(A.lmeta + b);
    if (lane < kLowCap) ent = __ldcg(A.lent + (size_t)b * kLowCap + lane);
    rmin = (uint32_t)__ldcg(rowmin + b);
    // every member has read b's state before the lead can update it
    team_sync(tm);
  }
  uint32_t target = yb - 1;
  int start = 0;
  bool fresh = true;  // b came from the free list (owns its low-set cache)
  uint32_t mnw = 0xffffffffu;
  bool track_min = false, dirty = false;
  LowBuild lb;
  bool walk = meta.y > 0 && target <= (uint32_t)meta.x;
  bool skip = false;
  if (!walk) {
    if (rmin > target) {
      skip = true;  // row min too high: no admissible edge (min only grows)
      OTPRG_STAT(6);
    } else {  // full scan from position 0 (rebuilding the low set in warp mode)
      OTPRG_STAT(5);
      track_min = true;
      if (!kTail && tm.size == 1) {
        meta = make_int4((int)(target + kLowLevels), 0, 0, 0);
        lb.on = true;
        lb.cnt = 0;
        lb.up_rep = S::rep(target + kLowLevels);
        lb.ent = A.lent + (size_t)b * kLowCap;
        dirty = true;
      }
    }
  }
  bool scanning = !walk && !skip;

  while (true) {
    int a = -1;
    if (walk) {
      const int pos = (int)(uint32_t)ent;
      const uint32_t kv = (uint32_t)(ent >> 32);
      const bool ok = lane < meta.z && pos >= start && kv + (uint32_t)tp[pos] == target;
      const unsigned bal = __ballot_sync(kFull, ok);
      if (lead) ++walks;
      if (bal) {
        a = __shfl_sync(kFull, pos, __ffs(bal) - 1);
        OTPRG_STAT(2);
      } else if (meta.y >= lda) {
        OTPRG_STAT(3);
      } else {  // cache covers [0, cov) only: scan the rest
        OTPRG_STAT(4);
        walk = false;
        scanning = true;
        start = max(start, meta.y);
        if (!kTail && tm.size == 1 && meta.z < kLowCap && start == meta.y) {  // extend the cache
          lb.on = true;
          lb.cnt = meta.z;
          lb.up_rep = S::rep((uint32_t)meta.x);
          lb.ent = A.lent + (size_t)b * kLowCap;
          dirty = true;
        }
      }
    }
    if (scanning) {
      const unsigned long long ts0 = acc ? globaltimer() : 0;
      a = warp_scan<T, kSmem, kMid ? OTPRG_MID_UNROLL : (kTail ? OTPRG_TAIL_UNROLL : kUnrollSmem)>(kT + (size_t)b * lda, tp, lda, start,
                                                                       target, track_min, mnw, lb,
                              lane, tm, bytes);
      if (acc) acc[0] += globaltimer() - ts0;
      if (lead) ++steps;
      if (dirty) {
        meta.z = lb.cnt;
        meta.y = lb.full_pos >= 0 ? lb.full_pos + 1 : (a >= 0 ? a + 1 : lda);
        if (lb.full_pos >= 0) lb.on = false;
      }
#ifdef OTPRG_DEBUG_SCAN
      if (lead) {  // serial re-check of the warp scan
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
      // (clamped into int: a uint32 pad sum 0xffffffff must not read as -1)
      if (track_min)
        m = (uint32_t)team_min(tm, (int)min(__reduce_min_sync(kFull, S::hmin(mnw)), 0x7fffffffu), lane);
      if (lead) {
        if (track_min) rowmin[b] = (T)m;
        if (fresh && dirty) A.lmeta[b] = meta;
        if (yb + 1 > tmax) report(ctl, 11, (int)phase, b, (int)yb);
        A.yb[b] = (int32_t)(yb + 1);
        P.list_out[slot] = b;
        P.mp_out[slot] = make_int2(-1, -1);
        atomicAdd(P.cnt_out, 1);  // results unused: compiled to fire-and-forget reductions
        atomicAdd(P.exh_out, 1);
      }
      if (in_slot >= 0) {  // b proposes again next phase from the same slot
        // (a displaced b continuing here: its cache may be written this
        // phase by its own chain, not in this warp's registers -> reload)
        nx.ok = fresh;
        nx.b = b;
        nx.yb = yb + 1;
        nx.rowmin = track_min ? (uint32_t)(T)m : rmin;
        nx.meta = meta;
        nx.ent = ent;
        if (fresh && dirty) {  // entries rewritten by this warp's lanes
          __syncwarp();
          nx.ent = lane < kLowCap ? __ldcg(A.lent + (size_t)b * kLowCap + lane) : 0ull;
        }
      }
      return;
    }
    const unsigned long long key = ((unsigned long long)cur_tag << 32) | (uint32_t)b;
    unsigned long long old = 0, hp = 0;
    int ma = -1;
    OTPRG_STAT(7);
    if (acc && lead) acc[2] += 1;  // proposals of this warp's chains (timeline)
    const unsigned long long ta0 = acc ? globaltimer() : 0;
    if (lead) {
      old = atomicMin(H + a, key);
      // the partner lookup of a first take, issued with the atomic (both
      // arrays are stable for entries it uses: see below)
      hp = __ldcg(Hprev + a);
      ma = __ldcg(A.match_a + a);
    }
    old = team_bcast(tm, old, lane);
    if (acc) acc[1] += globaltimer() - ta0;
    const uint32_t old_tag = (uint32_t)(old >> 32);
#ifdef OTPRG_DEBUG_SCAN
    if (lead && old_tag < cur_tag)  // key from a later phase
      report(ctl, 13, (int)phase, b, a, (int)~old_tag, (int)(uint32_t)old);
#endif
    if (old < key) {  // a is held by a lower b of this phase: next candidate
      start = a + 1;
      continue;
    }
    if (lead && fresh && dirty) A.lmeta[b] = meta;
    if (old_tag == cur_tag) {  // displaced b2 continues after a (plain scan)
      b = (int)(uint32_t)old;
      OTPRG_STAT(1);
      yb = (uint32_t)__ldcg(A.yb + b);
      target = yb - 1;
      start = a + 1;
      fresh = false;
      walk = false;
      scanning = true;
      track_min = false;
      dirty = false;
      lb.on = false;
      continue;
    }
    int partner = -1;
    if (lead) {
      // a is taken for the first time this phase: its partner before this
      // phase is displaced (it is freed by apply_phase).  If a was matched in
      // the previous phase, that partner is the previous phase's winner (the
      // global matching is being updated concurrently in this phase);
      // otherwise match_a, which is complete for all earlier phases (the
      // apply of M'_{phase-1} only writes match_a of a in M'_{phase-1}).
      partner = (uint32_t)(hp >> 32) == prev_tag ? (int)(uint32_t)hp : ma;
      if (partner >= 0) {
        atomicAdd(P.cnt_out, 1);
      }
      P.list_out[slot] = partner;  // -1: a hole in the next list
      P.mp_out[slot] = make_int2(a, partner);
      atomicAdd(P.mp_cnt_out, 1);
    }
    if (in_slot >= 0) {  // the displaced partner proposes next phase from this slot
      partner = (int)team_bcast(tm, (unsigned long long)(unsigned)partner, lane);
      nx.ok = true;
      nx.b = partner;
      if (partner >= 0) {  // matched since an earlier phase: its state is stable
        nx.yb = (uint32_t)__ldcg(A.yb + partner);
        nx.meta = __ldcg(A.lmeta + partner);
        nx.ent = lane < kLowCap ? __ldcg(A.lent + (size_t)partner * kLowCap + lane) : 0ull;
        nx.rowmin = (uint32_t)__ldcg(rowmin + partner);
      }
    }
    return;
  }
}

// kTail: the same loop specialised for small phases (every chain run by a
// team): no streaming list build, no low-set construction in the scans (only
// warp-mode chains build caches), so less live state and code.  The full
// loop stops at the first phase small enough for teams of 8 when A.tail_switch
// is set, and the tail launch continues from there (multi-launch state as
// for the stepping API: bar_base, applied).
template <typename T, bool kSmem, bool kTail, int kMid = 0>
__global__ void __launch_bounds__(kBlock, 1) phase_loop_kernel(SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s_t = reinterpret_cast<T*>(smem_raw);
  Ctl* ctl = A.ctl;
  const int lda = ctl->lda;
  const int n_b = ctl->n_b;
  const int thresh = ctl->thresh;
  const uint32_t cap = (uint32_t)ctl->phase_cap;
  const uint32_t tmax = ctl->tmax;
  // Read once at launch; ctl->phase / ctl->applied are only written after
  // this launch's first grid barrier, so late-starting blocks read the same.
  uint32_t phase = ld_cg(reinterpret_cast<const unsigned*>(&ctl->phase));
  const uint32_t applied0 = ld_cg(reinterpret_cast<const unsigned*>(&ctl->applied));
  const int lane = threadIdx.x & 31;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long bytes = 0, steps = 0, walks = 0;
  T* tg = static_cast<T*>(A.t);
  // Barrier targets: the arrival count at launch is ctl->bar_base (written by
  // the previous launch at exit); every barrier adds gridDim.x.
  unsigned bar_target = ld_cg(reinterpret_cast<const unsigned*>(&ctl->bar_base));
  const int warps_per_block = blockDim.x >> 5;
  const int total_warps = gridDim.x * warps_per_block;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int gthreads = gridDim.x * blockDim.x;

  if constexpr (kSmem) {  // global t is complete at launch (previous launch applied its M')
    const uint4* src = reinterpret_cast<const uint4*>(tg);
    uint4* dst = reinterpret_cast<uint4*>(s_t);
    const int nvec = lda * (int)sizeof(T) / 16;
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = __ldcg(src + i);
  }
  __shared__ int s_ctl[5];
  __shared__ unsigned long long s_team[kBlock / 32][10];  // team broadcast slots
  __shared__ unsigned s_stat[8];
  if (threadIdx.x < 8) s_stat[threadIdx.x] = 0;
  bool first = true;
  int n_prev = -1;
  int tsize_prev = 1;  // team size of the previous phase: guess for the prefetch
  const int wib = threadIdx.x >> 5;
  const int n_a = ctl->n_a;
  // Global part of apply M'_p (matching, global t), entries striped over the
  // blocks (entry q = thread * grid + block).  The first entry of every
  // thread is loaded speculatively at the top, in the same round trips as
  // the phase counters and the chain prologue; only its stores wait.
  auto apply_global = [&](const int2* mp_prev, const unsigned long long* Hq, int m_slots,
                          uint32_t ph, int q0, int2 e0, int b0, uint32_t t0) {
    for (int i = q0; i < m_slots; i += gthreads) {
      int2 e;
      int b;
      uint32_t nt;
      if (i == q0) {
        e = e0;
        b = b0;
        nt = t0 + 1u;
      } else {
        e = __ldcg(mp_prev + i);
        if (e.x < 0) continue;  // slot of an exhausted chain
        b = (int)(uint32_t)__ldcg(Hq + e.x);
        nt = (uint32_t)__ldcg(tg + e.x) + 1u;
      }
      const int a = e.x, old_b = e.y;
      if (a < 0) continue;
      if (old_b >= 0) A.match_b[old_b] = -1;
      A.match_a[a] = b;
      A.match_b[b] = a;
      if (nt > tmax) report(ctl, 12, (int)ph, a, (int)nt);
      tg[a] = (T)nt;
    }
  };
  const int q0 = (int)threadIdx.x * (int)gridDim.x + (int)blockIdx.x;
  // This warp's first proposer of the coming phase: prefetched at the top,
  // or (after a static-slot phase) carried over from the chain that produced it.
  Prefetch pf;
  pf.ok = false;
  pf.i = -1;
  bool prev_static = false;  // the previous phase wrote its outputs to static slots
  while (true) {
    const int r_prev = phase % 3, r_cur = (phase + 1) % 3, r_nxt = (phase + 2) % 3;
    // apply M'_{phase} unless the previous launch already did
    const bool apply = phase > 0 && !(first && applied0 == phase);
    const int32_t* list_in = r_prev == 0 ? A.list[0] : (r_prev == 1 ? A.list[1] : A.list[2]);
    const int2* mp_prev = A.mp[0];
    if (r_prev == 1) mp_prev = A.mp[1];
    if (r_prev == 2) mp_prev = A.mp[2];
    const unsigned long long* Hq = (phase & 1) ? A.holder[1] : A.holder[0];  // phase's winners
    if (threadIdx.x == 0) {  // one read per block, broadcast: uniform branches
      s_ctl[0] = ld_cg(&ctl->status);
      s_ctl[1] = ld_cg(&ctl->cnt[r_prev]);
      s_ctl[2] = apply ? ld_cg(&ctl->mp_cnt[r_prev]) : 0;
      s_ctl[3] = ld_cg(&ctl->exh[r_prev]);
      s_ctl[4] = ld_cg(&ctl->slots[r_prev]);
    }
    // Speculative loads in the same round trip as the counters: this warp's
    // first proposer of the coming phase (static index under the previous
    // team size; b is clamped, used only if the index is < n) and its chain
    // prologue, and this thread's M' entry.
    if (!prev_static) {  // (else pf holds the carry: same team size and slot)
      pf.i = (wib / tsize_prev) * (int)gridDim.x + (int)blockIdx.x;
      pf.ok = pf.i < n_b;
    }
    if (!prev_static && pf.ok) {
      pf.b = __ldcg(list_in + pf.i);  // may be a hole (-1)
      const int bb = min(max(pf.b, 0), n_b - 1);
      pf.yb = (uint32_t)__ldcg(A.yb + bb);
      pf.meta = __ldcg(A.lmeta + bb);
      pf.ent = lane < kLowCap ? __ldcg(A.lent + (size_t)bb * kLowCap + lane) : 0ull;
      pf.rowmin = (uint32_t)__ldcg(static_cast<const T*>(A.rowmin) + bb);
    }
    int mp_a = -1;
    if (kSmem && apply && (int)threadIdx.x < n_b) mp_a = __ldcg(&mp_prev[threadIdx.x].x);
    int2 g_e = make_int2(0, -1);
    int g_b = 0;
    uint32_t g_t = 0;
    if (apply && q0 < n_b) {
      g_e = __ldcg(mp_prev + q0);  // may be a hole (a = -1)
      const int a = min(max(g_e.x, 0), n_a - 1);
      g_b = (int)(uint32_t)__ldcg(Hq + a);
      g_t = (uint32_t)__ldcg(tg + a);
    }
    __syncthreads();
    const int status = s_ctl[0], n = s_ctl[1], m_prev = s_ctl[2], x_prev = s_ctl[3];
    const int n_slots = s_ctl[4];  // slots of list_in / mp_prev (holes are -1)
    __syncthreads();
    if (leader && !first) {
      ctl->phase = phase;  // published only after a grid barrier of this launch
      // conservation: every proposer of B' either holds an a or ended free
      if (x_prev + m_prev != n_prev) report(ctl, 7, (int)phase, n_prev, m_prev, x_prev);
    }
    first = false;

    // ---- apply M'_{phase}: shared t (every block) and the global state ----
    if (m_prev > 0) {
      if constexpr (kSmem) {
        for (int i = threadIdx.x; i < n_slots; i += blockDim.x) {
          const int a = i < n_b && i == (int)threadIdx.x ? mp_a : __ldcg(&mp_prev[i].x);
          if (a >= 0) s_t[a] = (T)(s_t[a] + 1);  // each a appears once
        }
      }
      apply_global(mp_prev, Hq, n_slots, phase, q0, g_e, g_b, g_t);
      if (leader) ctl->applied = phase;
    }
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
    if (!kTail && A.tail_switch && n_slots * (OTPRG_MID ? 4 : 8) <= total_warps * OTPRG_TEAM_OVERSUB / OTPRG_TEAM_DEN)
      break;  // the tail launch(es) take over from this phase
    if constexpr (kMid != 0) {
      if (n_slots * 8 <= total_warps * OTPRG_TEAM_OVERSUB / OTPRG_TEAM_DEN) break;  // teams of 8 from here
    }
    phase += 1;
    n_prev = n;
    // Barriers only in iterations that run a phase, so every executed phase
    // passes exactly kBarriers of them (bar_target is derived from that).
    if constexpr (!kSmem) {  // P reads global t: the apply must be complete
      bar_target += gridDim.x;
      grid_barrier(ctl, bar_target);
    }
#ifdef OTPRG_DEBUG_SCAN
    bar_target += gridDim.x;
    grid_barrier(ctl, bar_target);
    if (blockIdx.x == 0 && phase > 0) {  // full state consistency before the phase
      __shared__ int s_free, s_bad;
      if (threadIdx.x == 0) s_free = 0, s_bad = -1;
      __syncthreads();
      for (int b = threadIdx.x; b < ctl->n_b; b += blockDim.x) {
        const int a = __ldcg(A.match_b + b);
        if (a == -1) atomicAdd(&s_free, 1);
        else if (__ldcg(A.match_a + a) != b) atomicMax(&s_bad, b);
      }
      __syncthreads();
      if (threadIdx.x == 0 && (s_free != n || s_bad >= 0))
        report(ctl, 10, (int)phase, n, s_free, s_bad);
      __syncthreads();
    }
#endif
    // Timeline slots (ns): 0 phase start, 1 apply done (block 0), 2/3 last /
    // first block done with P (3 stores ~t), 4 after the barrier, 7 n_i.
    unsigned long long* tr =
        (A.trace && phase <= A.trace_cap) ? A.trace + (size_t)(phase - 1) * kTraceSlots : nullptr;
    if (leader) {
      A.free_counts[phase - 1] = n;
      // (a reduction, not a load + store: block 0 must not wait a round trip here)
      atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->sum_ni), (unsigned long long)n);
      ctl->cnt[r_nxt] = 0;  // r_nxt was last read at the top of phase - 1
      ctl->mp_cnt[r_nxt] = 0;
      ctl->work[r_nxt] = 0;
      ctl->exh[r_nxt] = 0;
      ctl->slots[r_nxt] = 0;
      if (tr) tr[0] = globaltimer(), tr[7] = (unsigned long long)n;
    }
    const T* tp = kSmem ? s_t : tg;

    // ---- P step: proposal chains over the free list of phase `phase` ----
    PhasePtrs P;
    P.list_out = r_cur == 0 ? A.list[0] : (r_cur == 1 ? A.list[1] : A.list[2]);
    P.mp_out = r_cur == 0 ? A.mp[0] : (r_cur == 1 ? A.mp[1] : A.mp[2]);
    P.cnt_out = &ctl->cnt[r_cur];
    P.mp_cnt_out = &ctl->mp_cnt[r_cur];
    P.exh_out = &ctl->exh[r_cur];
    P.slot_out = &ctl->slots[r_cur];
    // Team size for this phase: few proposers -> several warps per row
    // (uniform over the grid since n is).  First proposer of every team is
    // static, striped across blocks; the rest are grabbed from a counter.
    int tsize = 1;  // (proposers are assigned by slot: size by the slot count)
    if (kTeams) {
      const int tw = total_warps * OTPRG_TEAM_OVERSUB / OTPRG_TEAM_DEN;  // (team size vs the warps)
      if (n_slots * 8 <= tw) tsize = 8;
      else if (n_slots * 4 <= tw) tsize = 4;
      else if (n_slots * 2 <= tw) tsize = 2;
    }
    if constexpr (kTail && OTPRG_TAIL_CONST) {
      // the tail starts at a phase with teams of 8 and the slot count never
      // grows: a compile-time team size (and one slot per team)
      if (tsize != (kMid ? kMid : 8)) {
        if (leader) report(ctl, 14, (int)phase, n_slots);
        break;
      }
      tsize = kMid ? kMid : 8;
    }
    // (phase 1's lists come from the streaming propose kernel when it ran)
    const bool bulk = !kTail && kBulk && n >= total_warps && !(phase == 1 && A.pre_scanned);
    if (bulk) {
      // Large phase: first stream every proposer's row once at full HBM
      // bandwidth (warps in flight, no dependent atomics), recording its
      // admissible positions (level 0 of the low-set cache) and row minimum;
      // the chains below then mostly walk these lists.
      Team solo{1, 0, 0u, s_team[wib]};
      for (int q = wib * (int)gridDim.x + (int)blockIdx.x; q < n_slots; q += total_warps) {
        const int b = __ldcg(list_in + q);
        if (b < 0) continue;
        const uint32_t target = (uint32_t)__ldcg(A.yb + b) - 1u;
        const int4 meta0 = __ldcg(A.lmeta + b);
        if (meta0.y >= lda && target <= (uint32_t)meta0.x) continue;  // complete & valid
        LowBuild lb;
        lb.on = true;
        lb.up_rep = Simd<T>::rep(target);
        lb.ent = A.lent + (size_t)b * kLowCap;
        uint32_t mnw = 0xffffffffu;
        warp_scan<T, kSmem>(static_cast<const T*>(A.kT) + (size_t)b * lda, tp, lda, 0, target, true,
                            mnw, lb, lane, solo, bytes, true);
        const uint32_t m = __reduce_min_sync(kFull, Simd<T>::hmin(mnw));
        if (lane == 0) {
          A.lmeta[b] = make_int4((int)target, lb.full_pos >= 0 ? lb.full_pos + 1 : lda, lb.cnt, 0);
          static_cast<T*>(A.rowmin)[b] = (T)m;
        }
      }
      bar_target += gridDim.x;
      grid_barrier(ctl, bar_target, tr ? tr + 9 : nullptr);
      if (tr && leader) tr[8] = globaltimer();
    }
    const int tib = wib / tsize;  // team index in the block
    Team tm{tsize, wib % tsize, 1u + (unsigned)tib, s_team[tib]};
    const int teams_per_block = warps_per_block / tsize;
    const int total_teams = gridDim.x * teams_per_block;
    int i = tib * (int)gridDim.x + (int)blockIdx.x;
    unsigned long long acc[3] = {0ull, 0ull, 0ull};
    const unsigned long long steps0 = steps, walks0 = walks;
    const unsigned long long tp0 = tr ? globaltimer() : 0;
    const bool had_work = i < n_slots;
    // The prefetched prologue is current unless the bulk build rewrote it.
    // All warps of a team must take their prologue from the same place (a
    // team's lead may update Y(b) / the cache of b before a late member
    // reads them), hence the same-team-size condition.
    bool use_pf = pf.ok && !bulk && i == pf.i && tsize == tsize_prev;
    const bool single = n_slots <= total_teams;  // every team has at most its static slot
    // Static slots for the outputs of this phase: every team has at most its
    // slot, few holes (the slot range is not compacted), same team size next
    // phase (it depends on the slot count only).
    const bool static_out = kStatic && kSmem && single && !bulk && (n_slots - n) * OTPRG_STATIC_HOLES <= n_slots;
    if (static_out && leader) ctl->slots[r_cur] = n_slots;
    tsize_prev = tsize;
    pf.ok = false;  // (from here on: the carry for the next phase)
    pf.i = i;
    while (i < n_slots) {
      const int b = use_pf ? pf.b : __ldcg(list_in + i);
      if (b >= 0) {
        run_chain<T, kSmem, kTail, kMid>(b, A, P, tp, lda, phase, tmax, lane, bytes, steps, walks, s_stat,
                            tr ? acc : nullptr, tm, pf, use_pf, static_out ? i : -1, pf);
      } else if (static_out) {  // a hole stays a hole
        if (lane == 0 && tm.rank == 0) {
          P.list_out[i] = -1;
          P.mp_out[i] = make_int2(-1, -1);
        }
        pf.ok = true;
        pf.b = -1;
      }
      use_pf = false;
      if (single || (kTail && OTPRG_TAIL_CONST)) break;
      unsigned long long nx = 0;
      if (lane == 0 && tm.rank == 0) nx = (unsigned long long)(total_teams + atomicAdd(&ctl->work[r_cur], 1));
      i = (int)team_bcast(tm, nx, lane);
    }
    if (tr && had_work && lane == 0) {  // slowest warp: scan / atomic / total ns
      atomicMax(tr + 1, acc[0]);
      atomicMax(tr + 5, acc[1]);
      atomicMax(tr + 6, globaltimer() - tp0);
      // chain structure maxima over warps: row scans, cache walks, proposals
      atomicMax(tr + 10, steps - steps0);
      atomicMax(tr + 11, walks - walks0);
      atomicMax(tr + 12, acc[2]);
    }
    prev_static = static_out;
    bar_target += gridDim.x;
    grid_barrier(ctl, bar_target, tr ? tr + 2 : nullptr, tr ? tr + 3 : nullptr);
    if (tr && leader) tr[4] = globaltimer();
  }
  if (leader) ctl->bar_base = bar_target;  // every block exits with the same count
  if (lane == 0 && (bytes | steps | walks)) {
    atomicAdd(&ctl->bytes_touched, bytes);
    atomicAdd(&ctl->chain_steps, steps);
    atomicAdd(&ctl->list_walks, walks);
  }
  __syncthreads();
  if (threadIdx.x < 8 && s_stat[threadIdx.x])
    atomicAdd(&ctl->stat[threadIdx.x], (unsigned long long)s_stat[threadIdx.x]);
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
      A.holder[0][i] = ~0ull;
      A.holder[1][i] = ~0ull;
    }
    if (i < n_b) {
      A.match_b[i] = -1;
      A.yb[i] = 1;  // init_state: Y(b) = 1, Y(a) = 0 (assignment.cpp:54-60)
      rowmin[i] = 0;
      A.lmeta[i] = make_int4(0, 0, 0, 0);
      A.list[0][i] = i;  // phase 1 proposes every b
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

template <typename T, bool kSmem, bool kTail, int kMid = 0>
void* loop_fn() {
  return reinterpret_cast<void*>(&phase_loop_kernel<T, kSmem, kTail, kMid>);
}

// tail: 0 the full loop, 4 the mid loop (teams of 4), 8 the tail loop (teams of 8)
void* pick_loop(int width, bool smem_t, int tail = 0) {
  return with_width(width, [&](auto tag) {
    using T = decltype(tag);
    if (tail == 4) return loop_fn<T, true, true, 4>();
    if (tail) return loop_fn<T, true, true>();
    return smem_t ? loop_fn<T, true, false>() : loop_fn<T, false, false>();
  });
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
    smem_attr_raise(fn, smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem) != cudaSuccess)
    return 0;
  return per_sm * num_sms;
}

// Whether the tail-specialised loop can follow the full one on `grid` blocks.
static bool tail_usable(int width, bool smem_t, int lda, int grid, int ts = 8) {
  if (!OTPRG_TAIL || !smem_t) return false;
  if (OTPRG_MID && ts == 8 && !tail_usable(width, smem_t, lda, grid, 4)) return false;  // (both or neither)
  void* fn = pick_loop(width, true, ts);
  const size_t smem = phase_loop_smem(width, true, lda);
  if (smem > 48 * 1024) smem_attr_raise(fn, smem);
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem) != cudaSuccess) return false;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms >= grid;
}

int phase_loop_launches(int width, bool smem_t, int lda, int grid) {
  return tail_usable(width, smem_t, lda, grid) ? (OTPRG_MID ? 3 : 2) : 1;
}

cudaError_t launch_phase_loop(const SolveArgs& a, int width, bool smem_t, int lda, int grid,
                              cudaStream_t s) {
  const bool tail = tail_usable(width, smem_t, lda, grid);
  SolveArgs args = a;
  args.tail_switch = tail ? 1 : 0;
  void* params[] = {&args};
  const size_t smem = phase_loop_smem(width, smem_t, lda);
  cudaError_t e = cudaLaunchCooperativeKernel(pick_loop(width, smem_t), dim3(grid), dim3(kBlock), params, smem, s);
  if (e != cudaSuccess || !tail) return e;
  // (a solve that already ended returns at the tail's first top)
  if (OTPRG_MID) {
    e = cudaLaunchCooperativeKernel(pick_loop(width, true, 4), dim3(grid), dim3(kBlock), params, smem, s);
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchCooperativeKernel(pick_loop(width, true, 8), dim3(grid), dim3(kBlock), params, smem, s);
}

cudaError_t launch_init_state(const SolveArgs& a, int n_a, int n_b, int lda, int width,
                              cudaStream_t s) {
  const int blocks = (lda + 255) / 256;
  with_width(width, [&](auto tag) {
    init_state_kernel<decltype(tag)><<<blocks, 256, 0, s>>>(a, n_a, n_b, lda);
    return 0;
  });
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
