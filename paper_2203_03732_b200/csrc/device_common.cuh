// device_common.cuh — shared device helpers for the sm_100a kernels:
// packed-SIMD traits for the rounded-cost entry types, L2-coherent loads for
// state that changes between phases, and a grid barrier for the persistent
// cooperative phase loop.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace otprg {

constexpr unsigned kFull = 0xffffffffu;

// Control block of one solve; lives in device memory, zero-initialised by the
// host before phase 1.  Fields written during the loop are only read through
// ld.cg / atomics (never through L1).
struct Ctl {
  // set by the host
  int32_t n_a, n_b, lda;
  int32_t thresh;       // floor(eps * min(n_a, n_b)) : stop when n_i <= thresh
  int32_t phase_cap;    // phase_bound(eps) + 8  (assignment.cpp:326)
  uint32_t tmax;        // storage bound on |Y| (type max - 2)
  // loop state
  uint32_t phase;       // phases executed so far
  uint32_t applied;     // last phase whose M' is applied to the global state
  int32_t cnt[3];       // free-b list sizes (rotating over phases)
  int32_t mp_cnt[3];    // first-held-a list sizes (rotating)
  int32_t work[3];      // dynamic proposer-grab counters (rotating)
  int32_t exh[3];       // b's that ended their chain unmatched (rotating)
  int32_t slots[3];     // output slots reserved (= chains run) per list (rotating)
  int32_t status;       // 0 ok, else otprg_status / device diagnostic code
  int32_t done;         // 1 once the termination test passed
  int32_t full_match;   // n_i == 0 at termination
  int64_t sum_ni;
  unsigned long long bytes_touched;
  unsigned long long chain_steps;
  unsigned long long list_walks;
  // chain statistics: 0 fresh chains, 1 takeovers, 2 proposals from the
  // low-set cache, 3 exhausted by a complete cache, 4 scans continuing past
  // the cache, 5 full rescans (cache rebuilt), 6 rowmin skips, 7 proposals
  unsigned long long stat[8];
  // %globaltimer span of the phase-1 propose scan (first block start, last warp end)
  unsigned long long prop_t0, prop_t1;
  // grid barrier (monotone arrival count)
  unsigned int bar_count;
  unsigned int bar_base;  // bar_count at the start of the next launch (written at exit)
  int32_t err[8];       // details of the first failure (written by its reporter only)
  // A-row-sharded rounds (shard_kernels.cu): the round state lives on the device so
  // the resident loop needs no host.  A round is (scan, exchange, DA[, top]).
  int32_t sh_mode;      // 0: first round of a phase (every free b), 1: rescan/resume of parked chains
  int32_t sh_nreq;      // requests (= chains) of the current round
  int32_t sh_park_cur;  // park buffer holding the current round's chains (mode 1)
  int32_t sh_rounds;    // refill rounds so far
  uint32_t sh_epoch;    // exchange rounds completed (the value peers' flags reach)
  int32_t sh_live;      // 1 while rounds remain (set by the ctl kernel at the end of a round)
};

#ifdef __CUDACC__
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned ld_cg(const unsigned* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long* p) {
  return __ldcg(p);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// scaled_floor (core.cpp:26-32): floor(c/eps), repaired so that
// RN(k*eps) <= c < RN((k+1)*eps).
__device__ __forceinline__ long long scaled_floor_dev(double c, double eps) {
  long long k = (long long)floor(__ddiv_rn(c, eps));
  while (__dmul_rn((double)(k + 1), eps) <= c) ++k;
  while (k > 0 && __dmul_rn((double)k, eps) > c) --k;
  return k;
}

// Records the first failure: only the thread that moves status from 0 writes
// the details, so they are never mixed between reporters.
__device__ __forceinline__ void report(Ctl* ctl, int code, int e0, int e1 = 0, int e2 = 0,
                                       int e3 = 0, int e4 = 0, int e5 = 0) {
  if (atomicCAS(&ctl->status, 0, code) == 0) {
    ctl->err[0] = e0; ctl->err[1] = e1; ctl->err[2] = e2;
    ctl->err[3] = e3; ctl->err[4] = e4; ctl->err[5] = e5;
  }
}

// Counting grid barrier.  ctl->bar_count only grows: the j-th barrier of a
// solve completes when it reaches j * gridDim.x, so each block derives its
// target from how many barriers it has passed (no reset, no last-arriver
// step; arrivals are fire-and-forget release reductions).  Requires all
// blocks co-resident (cooperative launch).  A wait longer than 4 s flags
// status 6 and returns instead of hanging the device.
__device__ __forceinline__ void grid_barrier(Ctl* ctl, unsigned target,
                                             unsigned long long* arrive_max = nullptr,
                                             unsigned long long* arrive_min_inv = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (arrive_max) {  // timeline: when this block finished its work
      const unsigned long long now = globaltimer();
      atomicMax(arrive_max, now);
      if (arrive_min_inv) atomicMax(arrive_min_inv, ~now);
    }
    // release (cumulative: covers the block's writes ordered by the
    // __syncthreads above) / acquire pair; no separate fences needed
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctl->bar_count) : "memory");
    if ((int)(ld_acquire(&ctl->bar_count) - target) < 0) {
      const unsigned long long t0 = globaltimer();
      while ((int)(ld_acquire(&ctl->bar_count) - target) < 0) {
        if (globaltimer() - t0 > 4000000000ull) {
          report(ctl, 6, (int)blockIdx.x);
          break;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---- mbarrier + 1-D TMA bulk copies (cp.async.bulk) -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Orders this thread's earlier generic-proxy shared-memory accesses before
// later async-proxy (bulk copy) writes to the same bytes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- packed SIMD traits over 32-bit words ---------------------------------
// sum = k + t saturating (never wraps to a small value), eq = per-element
// all-ones where sum == target, mn = per-element min.
template <typename T>
struct Simd;

template <>
struct Simd<uint8_t> {
  static constexpr int kEpw = 4;  // elements per 32-bit word
  static constexpr uint32_t kPadWord = 0xffffffffu;
  __device__ static uint32_t rep(uint32_t v) { return v * 0x01010101u; }
  __device__ static uint32_t add(uint32_t k, uint32_t t) { return __vaddus4(k, t); }
  __device__ static uint32_t eq(uint32_t s, uint32_t tg) { return __vcmpeq4(s, tg); }
  __device__ static uint32_t mn(uint32_t a, uint32_t b) { return __vminu4(a, b); }
  __device__ static uint32_t le(uint32_t s, uint32_t up) { return __vcmpleu4(s, up); }
  // per-element all-ones mask -> one bit per element (element 0 = bit 0)
  __device__ static uint32_t bits(uint32_t m) {
    return ((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u);
  }
  __device__ static uint32_t elem(uint32_t w, int i) { return (w >> (8 * i)) & 0xffu; }
  __device__ static uint32_t hmin(uint32_t w) {
    uint32_t m = min(w & 0xffu, (w >> 8) & 0xffu);
    return min(m, min((w >> 16) & 0xffu, w >> 24));
  }
};

template <>
struct Simd<uint16_t> {
  static constexpr int kEpw = 2;
  static constexpr uint32_t kPadWord = 0xffffffffu;
  __device__ static uint32_t rep(uint32_t v) { return v * 0x00010001u; }
  __device__ static uint32_t add(uint32_t k, uint32_t t) { return __vaddus2(k, t); }
  __device__ static uint32_t eq(uint32_t s, uint32_t tg) { return __vcmpeq2(s, tg); }
  __device__ static uint32_t mn(uint32_t a, uint32_t b) { return __vminu2(a, b); }
  __device__ static uint32_t le(uint32_t s, uint32_t up) { return __vcmpleu2(s, up); }
  __device__ static uint32_t bits(uint32_t m) { return ((m >> 15) & 1u) | ((m >> 30) & 2u); }
  __device__ static uint32_t elem(uint32_t w, int i) { return (w >> (16 * i)) & 0xffffu; }
  __device__ static uint32_t hmin(uint32_t w) { return min(w & 0xffffu, w >> 16); }
};

// One element per word (eps below ~1/65531: unit_floor beyond uint16).
template <>
struct Simd<uint32_t> {
  static constexpr int kEpw = 1;
  static constexpr uint32_t kPadWord = 0xffffffffu;
  __device__ static uint32_t rep(uint32_t v) { return v; }
  __device__ static uint32_t add(uint32_t k, uint32_t t) {
    const uint32_t s = k + t;
    return s < k ? 0xffffffffu : s;
  }
  __device__ static uint32_t eq(uint32_t s, uint32_t tg) { return s == tg ? 0xffffffffu : 0u; }
  __device__ static uint32_t mn(uint32_t a, uint32_t b) { return min(a, b); }
  __device__ static uint32_t le(uint32_t s, uint32_t up) { return s <= up ? 0xffffffffu : 0u; }
  __device__ static uint32_t bits(uint32_t m) { return m & 1u; }
  __device__ static uint32_t elem(uint32_t w, int) { return w; }
  __device__ static uint32_t hmin(uint32_t w) { return w; }
};

#endif  // __CUDACC__

// Largest representable entry of T: the pad value of kT rows, and the
// saturation value of k + t.  Targets are always strictly below it.
template <typename T>
__host__ __device__ constexpr uint32_t type_max() {
  return sizeof(T) == 1 ? 0xffu : sizeof(T) == 2 ? 0xffffu : 0xffffffffu;
}

// Calls f(T{}) with T the kT storage type of `width` bytes (1, 2 or 4).
template <typename F>
inline auto with_width(int width, F&& f) {
  if (width == 1) return f(uint8_t{});
  if (width == 2) return f(uint16_t{});
  return f(uint32_t{});
}

}  // namespace otprg
