// cost_kernels.cu — cost build + rounding into the compact B-major matrix
// kT[b][a] = k(a, b) = scaled_floor(c(a, b), eps) (reference
// scale_round_costs, src/core.cpp:34-53, with scaled_floor :26-32).
//
// All FP64 arithmetic uses explicit round-to-nearest intrinsics so no FMA
// contraction can change bits: the reference is built without
// -march and its cost formulas are plain IEEE double expressions.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

template <typename T>
__device__ __forceinline__ T clamp_store(long long k) {
  // k <= unit_floor < type max by construction of the storage choice.
  return (T)k;
}

// K1: dense row-major f64 cost[a][b] -> kT.  Unswapped (n_a >= n_b):
// kT[b][a] (32x32 smem transpose).  Swapped: internal rows are original a,
// so kT[a][b] is a straight row-major rounding.
template <typename T>
__global__ void round_dense_kernel(const double* __restrict__ cost, int n_a, int n_b,
                                   int swapped, double eps, T* __restrict__ kT, int lda,
                                   int* status) {
  __shared__ T tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (!swapped) {
    const int a0 = blockIdx.x * 32, b0 = blockIdx.y * 32;  // a along lda
    for (int r = ty; r < 32; r += 8) {
      const int a = a0 + r, b = b0 + tx;
      T v = (T)type_max<T>();
      if (a < n_a && b < n_b) {
        const double c = cost[(size_t)a * n_b + b];
        if (!(c >= 0.0 && c <= 1.0)) atomicCAS(status, 0, 2);
        else v = clamp_store<T>(scaled_floor_dev(c, eps));
      }
      tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int b = b0 + r, a = a0 + tx;
      if (b < n_b && a < lda) kT[(size_t)b * lda + a] = tile[tx][r];
    }
  } else {
    // internal (a' = b, b' = a): kT[a][b] = k(cost[a][b]); lda pads n_b.
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int r = ty; r < 32; r += 8) {
      const int a = r0 + r, b = c0 + tx;
      if (a >= n_a || b >= lda) continue;
      T v = (T)type_max<T>();
      if (b < n_b) {
        const double c = cost[(size_t)a * n_b + b];
        if (!(c >= 0.0 && c <= 1.0)) atomicCAS(status, 0, 2);
        else v = clamp_store<T>(scaled_floor_dev(c, eps));
      }
      kT[(size_t)a * lda + b] = v;
    }
  }
}

// K2 (exact-division form): 2-D points -> kT with c = sqrt(dx*dx + dy*dy) /
// sqrt(2) (gen_uniform_square, instances.cpp:70-75).  Internal orientation:
// pa are the n_ai demand points, pb the n_bi supply points; the formula is
// exactly symmetric under swapping the roles of the two points.  Used only
// when the threshold table below would not fit in shared memory
// (unit_floor > kThrSmemMax - 2, i.e. eps < 1/8190).
template <typename T>
__global__ void round_points_div_kernel(const double2* __restrict__ pa,
                                        const double2* __restrict__ pb, int n_ai, int n_bi,
                                        double eps, double sqrt2, T* __restrict__ kT, int lda) {
  for (int b = blockIdx.y; b < n_bi; b += gridDim.y) {
    const double2 q = pb[b];
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < lda; a += gridDim.x * blockDim.x) {
      T v = (T)type_max<T>();
      if (a < n_ai) {
        const double2 p = pa[a];
        const double dx = __dsub_rn(p.x, q.x);
        const double dy = __dsub_rn(p.y, q.y);
        const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        const double c = __ddiv_rn(__dsqrt_rn(d2), sqrt2);
        v = clamp_store<T>(scaled_floor_dev(c, eps));
      }
      kT[(size_t)b * lda + a] = v;
    }
  }
}

// K2 on the exact threshold table (otprg_points_threshold_table):
// k(a,b) = scaled_floor(sqrt(d2) / sqrt(2), eps) = max{j : thr[j] <= d2} with
// d2 = dx*dx + dy*dy in IEEE RN (the reference's bits up to the sqrt).
//
// Fast path, FP32 only: x_f = sqrt(dx_f^2 + dy_f^2) / (sqrt(2) eps) from
// float copies of the coordinates is within B of the real x = c / eps, B
// bounded on the host from the coordinates' magnitude and eps (`margin`).
// When x_f is more than margin (= 4 B) from its nearest integer, x is more
// than 3 B away from every integer, and then scaled_floor(c, eps) = floor(x)
// = floor(x_f) exactly (its division and repair steps move k only when x
// lies within a few ulps of an integer).  Lanes near a level boundary (a
// fraction ~2 margin of the elements: ~0.05 % at eps = 0.01 on the unit
// square) compute the exact FP64 d2 and walk the table in shared memory from
// floor(x_f) - 2 (<= k) upwards.  No FP64 sqrt or division anywhere, FP64 work only on
// the rare slow lanes; the fast path is ~12 FP32/INT/MUFU instructions per
// entry.  Every thread owns 16 B of a kT row (kV consecutive demand points,
// float copies in registers) and walks a strided set of supply rows, storing
// one 16-byte vector per row: the build is bound by issue and HBM writes.
constexpr int kThrSmemMax = 8192;
template <typename T>
struct K2Shape {
  // entries per thread (16 for u8 / u16, 8 for u32: one or two 16-byte
  // stores per row), entries per 32-bit word, words
  static constexpr int kV = sizeof(T) == 4 ? 8 : 16, kPer = 4 / sizeof(T), kW = kV / kPer;
};

// FP32 estimate of entry (a, b): z = x_f - 1/2, y = z + 1.5 * 2^23 (FP32):
// y's low bits are then rint(z) = floor(x_f), and |z - rint(z)| = 1/2 -
// (distance of x_f to the nearest integer), returned as the nearness.
__device__ __forceinline__ uint32_t k2_estimate(float px, float py, float qx, float qy, float inv_step,
                                                float& near) {
  const float dx = px - qx, dy = py - qy;
  const float z = fmaf(sqrt_approx(fmaf(dy, dy, dx * dx)), inv_step, -0.5f);
  const float y = __fadd_rn(z, 12582912.0f);
  near = fabsf(__fsub_rn(z, __fsub_rn(y, 12582912.0f)));
  return __float_as_uint(y);
}

// The exact level from FP64 d2 and the table, walking up from floor(x_f) - 2
// (<= the level: |x_f - x| < margin < 1).
__device__ __forceinline__ int k2_exact_level(double2 p, double2 q, uint32_t y, const double* thr, int uf) {
  const double ex = __dsub_rn(p.x, q.x), ey = __dsub_rn(p.y, q.y);
  const double d2 = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
  int k = max(0, min((int)(y - 0x4B400000u) - 2, uf));
  while (k < uf && thr[k + 1] <= d2) ++k;
  return k;
}

// The entries (b, a0 .. a0 + kV/2) that lie near a level boundary (nearness
// >= lim, a superset of the fast pass's test) get their exact level from
// FP64 d2 and the table, walking up from floor(x_f) - 2 (<= the level:
// |x_f - x| < margin < 1); single-element stores over the fast pass's row.
template <typename T>
__device__ __forceinline__ void k2_patch_half(const double2* __restrict__ pa, double2 q, int n_ai, int a0,
                                              const double* thr, int uf, float inv_step, float lim,
                                              T* __restrict__ out) {
  constexpr int kV = K2Shape<T>::kV;
  const float qx = __double2float_rn(q.x), qy = __double2float_rn(q.y);
  for (int j = 0; j < kV / 2 && a0 + j < n_ai; ++j) {
    const double2 p = pa[a0 + j];
    float near;
    const uint32_t y = k2_estimate(__double2float_rn(p.x), __double2float_rn(p.y), qx, qy, inv_step, near);
    if (near < lim) continue;
    out[j] = (T)k2_exact_level(p, q, y, thr, uf);
  }
}

// One chunk of rows of one thread: its block owns the contiguous supply rows
// [b_lo, b_hi), staged kK2Chunk at a time in shared memory as float points
// (one broadcast load per row).  Per row: the kV estimates (branch-free,
// independent: ILP across entries), one max of their nearness, the packed
// store.  A row with an entry within margin of a level boundary is queued as
// (b, a0) in this block's fix-up list and patched by round_points_fix_kernel
// after the build (inline when the list is full), so the fast loop never
// recomputes.  kPad: this thread's entries include pad columns (a >= n_ai),
// which hold the type maximum.
constexpr int kK2Chunk = 256;
#ifndef OTPRG_K2_PREFETCH
#define OTPRG_K2_PREFETCH 1
#endif
#ifndef OTPRG_K2_UNROLL
#define OTPRG_K2_UNROLL 1
#endif
constexpr int kK2Unroll = OTPRG_K2_UNROLL;
#ifndef OTPRG_K2_MINB
#define OTPRG_K2_MINB 1
#endif
template <typename T, bool kPad>
__device__ __forceinline__ void k2_chunk(const float2 (&pf)[K2Shape<T>::kV], const double2* __restrict__ pa,
                                         const double2* __restrict__ pb, int n_ai, int c0, int nr,
                                         const double* s_thr, const float2* s_q, int uf, float inv_step, float lim,
                                         float lim_patch, const uint32_t (&padw)[K2Shape<T>::kW],
                                         T* __restrict__ kT, int lda, int a0, uint2* fix, int fix_cap, int* s_fix) {
  constexpr int kV = K2Shape<T>::kV, kW = K2Shape<T>::kW;
  T* out = kT + (size_t)c0 * lda + a0;
  const float2* qp = s_q;
#if OTPRG_K2_PREFETCH
  float2 qn = qp[0];
#endif
#pragma unroll kK2Unroll
  for (int r = 0; r < nr; ++r, out += lda, ++qp) {
#if OTPRG_K2_PREFETCH
    const float2 q = qn;
    qn = qp[r + 1 < nr ? 1 : 0];  // the next row's point in flight during this row
#else
    const float2 q = *qp;
#endif
    uint32_t yv[kV];
    float dm[2] = {0.0f, 0.0f};  // nearness of each half of the entries
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      float nr_j;
      yv[j] = k2_estimate(pf[j].x, pf[j].y, q.x, q.y, inv_step, nr_j);
      dm[j / (kV / 2)] = fmaxf(dm[j / (kV / 2)], nr_j);
    }
    uint32_t w[kW];
    if constexpr (sizeof(T) == 1) {
#pragma unroll
      for (int q4 = 0; q4 < kW; ++q4)
        w[q4] = __byte_perm(__byte_perm(yv[4 * q4], yv[4 * q4 + 1], 0x0040),
                            __byte_perm(yv[4 * q4 + 2], yv[4 * q4 + 3], 0x0040), 0x5410);
    } else if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int q4 = 0; q4 < kW; ++q4) w[q4] = __byte_perm(yv[2 * q4], yv[2 * q4 + 1], 0x5410);
    } else {
#pragma unroll
      for (int q4 = 0; q4 < kW; ++q4) w[q4] = yv[q4] - 0x4B400000u;
    }
    if constexpr (kPad) {
#pragma unroll
      for (int q4 = 0; q4 < kW; ++q4) w[q4] |= padw[q4];
    }
#pragma unroll
    for (int v = 0; v < kW / 4; ++v)
      reinterpret_cast<uint4*>(out)[v] = make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
    if (fmaxf(dm[0], dm[1]) >= lim) {  // near a level boundary: patched after the build, or now
      const int br = c0 + r;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (dm[h] < lim) continue;
        const int ah = a0 + h * (kV / 2);
        const int slot = atomicAdd(s_fix, 1);
        if (slot < fix_cap) fix[slot] = make_uint2((uint32_t)br, (uint32_t)ah);
        else k2_patch_half<T>(pa, pb[br], n_ai, ah, s_thr, uf, inv_step, lim_patch, out + h * (kV / 2));
      }
    }
  }
}

// fix: per block (linear index) a count word in fix_cnt and fix_cap entries.
template <typename T>
__global__ void __launch_bounds__(256, OTPRG_K2_MINB) round_points_thr_kernel(const double2* __restrict__ pa,
                                                               const double2* __restrict__ pb,
                                                               int n_ai, int n_bi, const double* __restrict__ thr,
                                                               int thr_n, float inv_step, float margin,
                                                               T* __restrict__ kT, int lda, uint2* __restrict__ fix,
                                                               int* __restrict__ fix_cnt, int fix_cap,
                                                               float2* __restrict__ pa_f, float2* __restrict__ pb_f) {
  constexpr int kV = K2Shape<T>::kV, kPer = K2Shape<T>::kPer, kW = K2Shape<T>::kW;
  extern __shared__ __align__(16) double s_thr[];  // the threshold table (the inline patches)
  __shared__ float2 s_q[kK2Chunk];
  __shared__ int s_fix;
  for (int j = threadIdx.x; j < thr_n; j += blockDim.x) s_thr[j] = thr[j];
  if (threadIdx.x == 0) s_fix = 0;
  const int uf = thr_n - 2;  // unit_floor: thr[uf + 1] = +inf
  const float lim = 0.5f - margin;  // nearness >= lim: within margin of a level boundary
  const float lim_patch = lim - 1e-5f;  // the patch's test: a superset
  const int a0 = (blockIdx.x * blockDim.x + threadIdx.x) * kV;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  // this block's supply rows: a contiguous range
  const int per = (n_bi + gridDim.y - 1) / gridDim.y;
  const int b_lo = min(n_bi, (int)blockIdx.y * per), b_hi = min(n_bi, b_lo + per);
  float2 pf[kV];
#pragma unroll
  for (int j = 0; j < kV; ++j) {
    const double2 p = a0 + j < n_ai ? pa[a0 + j] : make_double2(0.0, 0.0);
    pf[j] = make_float2(__double2float_rn(p.x), __double2float_rn(p.y));
    if (blockIdx.y == 0 && a0 + j < n_ai) pa_f[a0 + j] = pf[j];  // (for the fix-up pass)
  }
  // pad entries (a >= n_ai) hold the type maximum
  uint32_t padw[kW];
#pragma unroll
  for (int q4 = 0; q4 < kW; ++q4) padw[q4] = 0u;
#pragma unroll
  for (int j = 0; j < kV; ++j)
    if (a0 + j >= n_ai) padw[j / kPer] |= type_max<T>() << (8 * sizeof(T) * (j % kPer));
  const bool active = a0 < lda, full = a0 + kV <= n_ai;
  uint2* my_fix = fix + (size_t)blk * fix_cap;
  for (int c0 = b_lo; c0 < b_hi; c0 += kK2Chunk) {
    const int nr = min(kK2Chunk, b_hi - c0);
    __syncthreads();  // (the previous chunk's points are consumed)
    for (int j = threadIdx.x; j < nr; j += blockDim.x) {
      const double2 q = pb[c0 + j];
      s_q[j] = make_float2(__double2float_rn(q.x), __double2float_rn(q.y));
      if (blockIdx.x == 0) pb_f[c0 + j] = s_q[j];
    }
    __syncthreads();
    if (!active) continue;
    if (full)
      k2_chunk<T, false>(pf, pa, pb, n_ai, c0, nr, s_thr, s_q, uf, inv_step, lim, lim_patch, padw, kT, lda, a0,
                         my_fix, fix_cap, &s_fix);
    else
      k2_chunk<T, true>(pf, pa, pb, n_ai, c0, nr, s_thr, s_q, uf, inv_step, lim, lim_patch, padw, kT, lda, a0,
                        my_fix, fix_cap, &s_fix);
  }
  __syncthreads();
  if (threadIdx.x == 0) fix_cnt[blk] = min(s_fix, fix_cap);
}

constexpr int kFixSlices = 8;
// The queued half rows: a thread per entry (half row, j) recomputes the
// estimate from the float copies and takes the exact level (FP64 d2 and the
// table) of the near ones, over the fast pass's store.
template <typename T>
__global__ void __launch_bounds__(256) round_points_fix_kernel(const double2* __restrict__ pa,
                                                               const double2* __restrict__ pb, int n_ai,
                                                               const double* __restrict__ thr, int thr_n,
                                                               float inv_step, float margin, T* __restrict__ kT,
                                                               int lda, const uint2* __restrict__ fix,
                                                               const int* __restrict__ fix_cnt, int fix_cap,
                                                               int blocks, const float2* __restrict__ pa_f,
                                                               const float2* __restrict__ pb_f) {
  constexpr int kH = K2Shape<T>::kV / 2;
  extern __shared__ __align__(16) double s_thr[];
  for (int j = threadIdx.x; j < thr_n; j += blockDim.x) s_thr[j] = thr[j];
  __syncthreads();
  const float lim_patch = 0.5f - margin - 1e-5f;
  const int uf = thr_n - 2;
  // kFixSlices blocks per main-kernel block (its list): latency-bound
  // dependent loads, so many threads in flight
  for (int w = blockIdx.x; w < blocks * kFixSlices; w += gridDim.x) {
    const int blk = w / kFixSlices, sl = w % kFixSlices;
    const int n = fix_cnt[blk] * kH;
    const uint2* f = fix + (size_t)blk * fix_cap;
    for (int e = sl * blockDim.x + threadIdx.x; e < n; e += kFixSlices * blockDim.x) {
      const uint2 ba = f[e / kH];
      const int a = (int)ba.y + e % kH;
      if (a >= n_ai) continue;
      const float2 pf = pa_f[a], qf = pb_f[ba.x];
      float nr;
      const uint32_t y = k2_estimate(pf.x, pf.y, qf.x, qf.y, inv_step, nr);
      if (nr < lim_patch) continue;
      kT[(size_t)ba.x * lda + a] = (T)k2_exact_level(pa[a], pb[ba.x], y, s_thr, uf);
    }
  }
}

// Range check of a point instance (AssignmentInstance::validate,
// core.cpp:15-21): the first (a, b) in the reference's row-major order whose
// cost sqrt(d2)/sqrt(2) is not in [0, 1] — d2 above d2_max (the largest d2
// with cost <= 1) or NaN — as atomicMin of a * n_b + b (original
// orientation).  Only launched when the host's bounding-box bound does not
// already prove every cost <= 1.
__global__ void points_range_kernel(const double2* __restrict__ pa, const double2* __restrict__ pb,
                                    int n_a, int n_b, double d2_max,
                                    unsigned long long* __restrict__ first) {
  for (int a = blockIdx.y; a < n_a; a += gridDim.y) {
    const double2 p = pa[a];
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < n_b; b += gridDim.x * blockDim.x) {
      const double2 q = pb[b];
      const double dx = __dsub_rn(p.x, q.x), dy = __dsub_rn(p.y, q.y);
      const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      if (!(d2 <= d2_max)) atomicMin(first, (unsigned long long)a * n_b + b);
    }
  }
}

// K3a: per-image normalisation of load_mnist_pair (instances.cpp:114-126):
// total = sum of the pixels (exact in double), pixel / total (IEEE RN).  One
// block per image.  A zero total is the reference's InputError (status 3).
__global__ void l1_normalize_kernel(const uint8_t* __restrict__ img, int count, int dim,
                                    double* __restrict__ out, int* status) {
  __shared__ unsigned s_sum;
  for (int i = blockIdx.x; i < count; i += gridDim.x) {
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    const uint8_t* src = img + (size_t)i * dim;
    unsigned part = 0;
    for (int p = threadIdx.x; p < dim; p += blockDim.x) part += src[p];
    atomicAdd(&s_sum, part);
    __syncthreads();
    const double total = (double)s_sum;  // integer sum < 2^53: exact, any order
    if (total == 0.0) {
      if (threadIdx.x == 0) atomicCAS(status, 0, 3);
    } else {
      for (int p = threadIdx.x; p < dim; p += blockDim.x)
        out[(size_t)i * dim + p] = __ddiv_rn((double)src[p], total);
    }
    __syncthreads();
  }
}

// K3b: all-pairs L1 / 2 with rounding (instances.cpp:134-142 then
// scale_round_costs).  c(a,b) = (sum_p |x_a[p] - y_b[p]|) / 2 summed in
// ascending p exactly like the reference (no reassociation, no FMA), so the
// bits match.  Block tile 64 a x 64 b, thread tile 4 x 4, pixels staged in
// shared memory in chunks of kP, p-major.
#ifndef OTPRG_L1_TA
#define OTPRG_L1_TA 8
#endif
#ifndef OTPRG_L1_TB
#define OTPRG_L1_TB 4
#endif
#ifndef OTPRG_L1_MINB
#define OTPRG_L1_MINB 2
#endif
constexpr int kL1TA = OTPRG_L1_TA, kL1TB = OTPRG_L1_TB;  // a / b entries per thread
#ifndef OTPRG_L1_P
#define OTPRG_L1_P 4
#endif
constexpr int kL1TileA = 16 * kL1TA, kL1TileB = 16 * kL1TB, kL1P = OTPRG_L1_P, kL1MaxList = 2048;

// Pixel-support masks: bit p of tile g's words is set when any image of the
// image tile g has pixel p != 0.  A pixel that is zero in every image of
// both tiles adds |0 - 0| = +0 to every sum of the block, which leaves the
// sum's bits unchanged (acc >= +0), so l1_round_kernel walks only the union
// of the two tiles' supports (config 3: about half the frame is empty).
__global__ void l1_tile_mask_kernel(const double* __restrict__ x, int n, int dim, int tiles, int rows,
                                    uint32_t* __restrict__ mask) {
  const int nw = (dim + 31) / 32;
  for (int g = blockIdx.x; g < tiles; g += gridDim.x) {
    const int r0 = g * rows, r1 = min(n, r0 + rows);
    for (int p0 = 0; p0 < nw * 32; p0 += blockDim.x) {
      const int p = p0 + threadIdx.x;
      bool any = false;
      if (p < dim)
        for (int r = r0; r < r1 && !any; ++r) any = x[(size_t)r * dim + p] != 0.0;
      const unsigned bal = __ballot_sync(kFull, any);
      if ((threadIdx.x & 31) == 0 && p < nw * 32) mask[(size_t)g * nw + (p >> 5)] = bal;
    }
  }
}

template <typename T, bool kStore = true>
__global__ void __launch_bounds__(256, OTPRG_L1_MINB) l1_round_kernel(const double* __restrict__ xa,
                                                       const double* __restrict__ yb, int n_ai,
                                                       int n_bi, int dim, double eps,
                                                       T* __restrict__ kT, int lda, int* status,
                                                       const uint32_t* __restrict__ mask_a,
                                                       const uint32_t* __restrict__ mask_b) {
  __shared__ __align__(16) double As[kL1P][kL1TileA];
  __shared__ __align__(16) double Bs[kL1P][kL1TileB];
  __shared__ short s_pl[kL1MaxList];  // ascending pixels in either tile's support
  __shared__ int s_np;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int a0 = blockIdx.x * kL1TileA, b0 = blockIdx.y * kL1TileB;
  const bool listed = mask_a != nullptr;  // (dim <= kL1MaxList)
  int np = dim;
  if (listed) {
    if (threadIdx.x < 32) {
      const int nw = (dim + 31) / 32;
      const uint32_t* ma = mask_a + (size_t)blockIdx.x * nw;
      const uint32_t* mb = mask_b + (size_t)blockIdx.y * nw;
      int base = 0;
      for (int w0 = 0; w0 < nw; w0 += 32) {
        const int w = w0 + (int)threadIdx.x;
        uint32_t m = w < nw ? (ma[w] | mb[w]) : 0u;
        const int c = __popc(m);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, inc, o);
          if ((int)threadIdx.x >= o) inc += y;
        }
        int pos = base + inc - c;
        while (m) {
          s_pl[pos++] = (short)(w * 32 + __ffs(m) - 1);
          m &= m - 1;
        }
        base += __shfl_sync(kFull, inc, 31);
      }
      if (threadIdx.x == 0) s_np = base;
    }
    __syncthreads();
    np = s_np;
  }
  double acc[kL1TA][kL1TB];
#pragma unroll
  for (int i = 0; i < kL1TA; ++i)
#pragma unroll
    for (int j = 0; j < kL1TB; ++j) acc[i][j] = 0.0;
  for (int p0 = 0; p0 < np; p0 += kL1P) {
    for (int e = threadIdx.x; e < max(kL1TileA, kL1TileB) * kL1P; e += blockDim.x) {
      const int r = e / kL1P, pp = e % kL1P, q = p0 + pp;
      const int p = q < np ? (listed ? (int)s_pl[q] : q) : -1;
      const int a = a0 + r, b = b0 + r;
      if (r < kL1TileA) As[pp][r] = (a < n_ai && p >= 0) ? xa[(size_t)a * dim + p] : 0.0;
      if (r < kL1TileB) Bs[pp][r] = (b < n_bi && p >= 0) ? yb[(size_t)b * dim + p] : 0.0;
    }
    __syncthreads();
    const int pend = min(kL1P, np - p0);
    for (int pp = 0; pp < pend; ++pp) {
      double av[kL1TA], bv[kL1TB];
#pragma unroll
      for (int i = 0; i < kL1TA; ++i) av[i] = As[pp][ty * kL1TA + i];
#pragma unroll
      for (int j = 0; j < kL1TB; ++j) bv[j] = Bs[pp][tx * kL1TB + j];
#pragma unroll
      for (int i = 0; i < kL1TA; ++i)
#pragma unroll
        for (int j = 0; j < kL1TB; ++j) acc[i][j] = __dadd_rn(acc[i][j], fabs(__dsub_rn(av[i], bv[j])));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kL1TA; ++i) {
    const int a = a0 + ty * kL1TA + i;
#pragma unroll
    for (int j = 0; j < kL1TB; ++j) {
      const int b = b0 + tx * kL1TB + j;
      if (b >= n_bi) continue;
      if (a < n_ai) {
        const double c = __ddiv_rn(acc[i][j], 2.0);
        if (!(c >= 0.0 && c <= 1.0)) {
          atomicCAS(status, 0, 2);  // core.cpp:18-21 rejects it (ParameterError)
          if (kStore) kT[(size_t)b * lda + a] = (T)type_max<T>();
        } else if (kStore) {
          kT[(size_t)b * lda + a] = clamp_store<T>(scaled_floor_dev(c, eps));
        }
      } else if (kStore && a < lda) {
        kT[(size_t)b * lda + a] = (T)type_max<T>();
      }
    }
  }
}

// Matched-pair L1/2 costs (load_mnist_pair's cost, instances.cpp:134-141, for
// matching_cost core.cpp:95-102): thread per original a, its partner's row,
// the pixel differences summed in ascending p (no FMA) exactly as K3.  self
// rows are xa (self_is_a) or yb; partners index the other side.
__global__ void l1_matched_cost_kernel(const double* __restrict__ xa, const double* __restrict__ yb, int dim,
                                       const int32_t* __restrict__ match, int n, int self_is_a,
                                       double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = match[i];
    if (j < 0) {
      out[i] = 0.0;
      continue;
    }
    const double* x = self_is_a ? xa + (size_t)i * dim : yb + (size_t)i * dim;
    const double* y = self_is_a ? yb + (size_t)j * dim : xa + (size_t)j * dim;
    double acc = 0.0;
    for (int p = 0; p < dim; ++p) acc = __dadd_rn(acc, fabs(__dsub_rn(x[p], y[p])));
    out[i] = __ddiv_rn(acc, 2.0);
  }
}

// Matched-pair point costs: x = this side's points, y = the other side's
// (the squared difference is symmetric, so either orientation gives the
// reference's bits for c(a, b)).
__global__ void points_matched_cost_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                           const int32_t* __restrict__ match, int n, double* __restrict__ out) {
  const double sqrt2 = __dsqrt_rn(2.0);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = match[i];
    if (j < 0) {
      out[i] = 0.0;
      continue;
    }
    const double dx = __dsub_rn(x[2 * (size_t)i], y[2 * (size_t)j]);
    const double dy = __dsub_rn(x[2 * (size_t)i + 1], y[2 * (size_t)j + 1]);
    out[i] = __ddiv_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))), sqrt2);
  }
}

__global__ void dense_matched_cost_kernel(const double* __restrict__ cost, int n_b,
                                          const int32_t* __restrict__ match, int n, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = match[i];
    out[i] = j < 0 ? 0.0 : cost[(size_t)i * n_b + j];
  }
}

// A given rounded-cost matrix (copy instances, ot.hpp:52-63): k[a][b]
// row-major int32 -> kT[b][a] (32x32 shared-memory transpose), pads = type max.
template <typename T>
__global__ void k_to_kT_kernel(const int32_t* __restrict__ k, int n_a, int n_b, T* __restrict__ kT,
                               int lda) {
  __shared__ T tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int a0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int r = ty; r < 32; r += 8) {
    const int a = a0 + r, b = b0 + tx;
    tile[r][tx] = (a < n_a && b < n_b) ? (T)k[(size_t)a * n_b + b] : (T)type_max<T>();
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, a = a0 + tx;
    if (b < n_b && a < lda) kT[(size_t)b * lda + a] = tile[tx][r];
  }
}

template <typename T>
__global__ void export_k_kernel(const T* __restrict__ kT, int n_ai, int n_bi, int lda,
                                int swapped, int32_t* __restrict__ k) {
  // original orientation row-major: unswapped k[a][b] = kT[b][a] (n_a = n_ai);
  // swapped k[a][b] = kT[a][b] with original n_a = n_bi, n_b = n_ai.
  const size_t total = (size_t)n_ai * n_bi;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    if (!swapped) {
      const size_t a = i / n_bi, b = i % n_bi;
      k[i] = kT[b * lda + a];
    } else {
      const size_t a = i / n_ai, b = i % n_ai;
      k[i] = kT[a * lda + b];
    }
  }
}

}  // namespace

cudaError_t launch_round_dense(const double* cost, int n_a, int n_b, bool swapped, double eps,
                               void* kT, int lda, int width, int* status, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid;
  if (!swapped)
    grid = dim3((lda + 31) / 32, (n_b + 31) / 32);
  else
    grid = dim3((lda + 31) / 32, (n_a + 31) / 32);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    round_dense_kernel<T><<<grid, block, 0, s>>>(cost, n_a, n_b, swapped, eps, static_cast<T*>(kT), lda, status);
    return 0;
  });
  return cudaGetLastError();
}

namespace {
// Bound on |x_f - x| (x = c / eps <= 1/eps + 1): float coordinates are off
// by <= C 2^-24 each (C = max |coordinate|), so dx_f, dy_f by <= 3 C 2^-24
// and d_f by <= 4.3 C 2^-24 + |d| 2^-22; x_f adds ~3 roundings (2^-22
// relative, the approximate sqrt included).  margin = 4 x that bound.
float k2_margin(double eps, double absmax) {
  const double xmax = 1.0 / eps + 1.0;
  const double bound = (4.3 * absmax * std::ldexp(1.0, -24) + std::sqrt(2.0) * std::ldexp(1.0, -22)) /
                           (std::sqrt(2.0) * eps) + xmax * std::ldexp(1.0, -21);
  return (float)std::min(0.5, 4.0 * bound + 1e-7);
}
constexpr int kK2MaxBlocks = 4096;
}  // namespace

size_t round_points_fix_bytes(int n_ai, int n_bi, int lda, int width, double eps, double absmax) {
  // twice the expected rows with an entry within margin of a boundary (a
  // full list only sends rows to the inline path), >= 1 M entries, <= 512 MB
  const int kv = width == 4 ? 8 : 16;
  const double m = k2_margin(eps, absmax);
  const double p_row = 1.0 - std::pow(std::max(0.0, 1.0 - 2.0 * m), kv / 2);  // (half rows)
  const double rows = 2.0 * n_bi * ((lda + kv - 1) / kv);
  const double want = std::min(64.0 * 1024 * 1024, std::max(1024.0 * 1024, 2.0 * rows * p_row + 65536.0));
  return 512 + (size_t)want * sizeof(uint2) + kK2MaxBlocks * sizeof(int) + ((size_t)n_ai + n_bi) * sizeof(float2) +
         64 * 1024;
}

cudaError_t launch_round_points2d(const double* pa, const double* pb, int n_ai, int n_bi,
                                  double eps, double sqrt2, const double* thr, int thr_n, double absmax,
                                  void* kT, int lda, int width, void* fix_buf, size_t fix_bytes, cudaStream_t s) {
  const double2* a2 = reinterpret_cast<const double2*>(pa);
  const double2* b2 = reinterpret_cast<const double2*>(pb);
  const size_t head = kK2MaxBlocks * sizeof(int) + ((size_t)n_ai + n_bi) * sizeof(float2);
  const size_t head_al = (head + 255) / 256 * 256;
  if (thr && thr_n >= 2 && thr_n <= kThrSmemMax && fix_buf && fix_bytes >= head_al + 64 * 1024) {
    // threads own kV entries of a row (16 for u8 / u16, 8 for u32); the grid
    // is one resident wave (occupancy-sized), contiguous supply row ranges
    // over grid.y
    const int kv = width == 4 ? 8 : 16;
    const int threads_x = (lda + kv - 1) / kv;
    const int bx = (threads_x + 255) / 256;
    const float inv_step = (float)(1.0 / (std::sqrt(2.0) * eps));
    const float margin = k2_margin(eps, absmax);
    const size_t smem = (size_t)thr_n * sizeof(double);
    // [per-block counts | float copies of the points | queued half rows]
    int* fix_cnt = static_cast<int*>(fix_buf);
    float2* pa_f = reinterpret_cast<float2*>(static_cast<char*>(fix_buf) + kK2MaxBlocks * sizeof(int));
    float2* pb_f = pa_f + n_ai;
    uint2* fix = reinterpret_cast<uint2*>(static_cast<char*>(fix_buf) + head_al);
    const size_t fix_total = (fix_bytes - head_al) / sizeof(uint2);
    with_width(width, [&](auto tag) {
      using T = decltype(tag);
      auto fn = round_points_thr_kernel<T>;
      auto fx = round_points_fix_kernel<T>;
      smem_attr_raise(fn, smem);
      smem_attr_raise(fx, smem);
      int per_sm = 0, dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
      int by = std::max(1, std::min(n_bi, sms * per_sm / bx));
      by = std::min(by, std::max(1, kK2MaxBlocks / bx));
      const int blocks = bx * by;
      const int cap = (int)std::min<size_t>(fix_total / blocks, (size_t)1 << 30);
      fn<<<dim3(bx, by), 256, smem, s>>>(a2, b2, n_ai, n_bi, thr, thr_n, inv_step, margin, static_cast<T*>(kT),
                                         lda, fix, fix_cnt, cap, pa_f, pb_f);
      fx<<<std::min(blocks * kFixSlices, 65535), 256, smem, s>>>(a2, b2, n_ai, thr, thr_n, inv_step, margin,
                                                      static_cast<T*>(kT), lda, fix, fix_cnt, cap, blocks, pa_f, pb_f);
      return 0;
    });
    return cudaGetLastError();
  }
  const int bx = (lda + 255) / 256;
  dim3 grid(bx < 8 ? bx : 8, n_bi < 65535 ? n_bi : 65535);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    round_points_div_kernel<T><<<grid, 256, 0, s>>>(a2, b2, n_ai, n_bi, eps, sqrt2, static_cast<T*>(kT), lda);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_points_range(const double* pa, const double* pb, int n_a, int n_b, double d2_max,
                                unsigned long long* first, cudaStream_t s) {
  const int bx = std::min(8, (n_b + 255) / 256);
  points_range_kernel<<<dim3(bx, std::min(n_a, 4096)), 256, 0, s>>>(
      reinterpret_cast<const double2*>(pa), reinterpret_cast<const double2*>(pb), n_a, n_b, d2_max, first);
  return cudaGetLastError();
}

cudaError_t launch_l1_normalize(const uint8_t* img, int count, int dim, double* out, int* status,
                                cudaStream_t s) {
  l1_normalize_kernel<<<count < 4096 ? count : 4096, 256, 0, s>>>(img, count, dim, out, status);
  return cudaGetLastError();
}

cudaError_t launch_l1_group_masks(const double* x, int n, int dim, int rows, uint32_t* mask, cudaStream_t s) {
  const int tiles = (n + rows - 1) / rows, nw = (dim + 31) / 32;
  if (tiles > 0)
    l1_tile_mask_kernel<<<std::min(tiles, 8192), std::min(1024, nw * 32), 0, s>>>(x, n, dim, tiles, rows, mask);
  return cudaGetLastError();
}

size_t l1_mask_bytes(int n_ai, int n_bi, int lda, int dim) {
  const int tiles = std::max(lda, n_ai) / kL1TileA + 1 + (n_bi + kL1TileB - 1) / kL1TileB;
  return (size_t)tiles * ((dim + 31) / 32) * sizeof(uint32_t);
}

namespace {
// masks of the A tiles (grid.x of them) and B tiles (grid.y); false when the
// walk goes over every pixel (dim beyond the list, or no mask buffer)
bool l1_masks(const double* xa, const double* yb, int n_ai, int n_bi, int dim, dim3 grid, uint32_t* masks,
              const uint32_t** ma, const uint32_t** mb, cudaStream_t s) {
  *ma = *mb = nullptr;
  if (!masks || dim > kL1MaxList) return false;
  const int nw = (dim + 31) / 32;
  uint32_t* b_masks = masks + (size_t)grid.x * nw;
  const int thr = std::min(1024, nw * 32);
  l1_tile_mask_kernel<<<std::min<int>(grid.x, 4096), thr, 0, s>>>(xa, n_ai, dim, grid.x, kL1TileA, masks);
  l1_tile_mask_kernel<<<std::min<int>(grid.y, 4096), thr, 0, s>>>(yb, n_bi, dim, grid.y, kL1TileB, b_masks);
  *ma = masks;
  *mb = b_masks;
  return true;
}
}  // namespace

cudaError_t launch_l1_round(const double* xa, const double* yb, int n_ai, int n_bi, int dim,
                            double eps, void* kT, int lda, int width, int* status,
                            cudaStream_t s, uint32_t* masks) {
  dim3 grid((lda + kL1TileA - 1) / kL1TileA, (n_bi + kL1TileB - 1) / kL1TileB);
  const uint32_t *ma, *mb;
  l1_masks(xa, yb, n_ai, n_bi, dim, grid, masks, &ma, &mb, s);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    l1_round_kernel<T><<<grid, 256, 0, s>>>(xa, yb, n_ai, n_bi, dim, eps, static_cast<T*>(kT), lda, status, ma,
                                            mb);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_l1_check(const double* xa, const double* yb, int n_ai, int n_bi, int dim, int* status,
                            cudaStream_t s, uint32_t* masks) {
  dim3 grid((n_ai + kL1TileA - 1) / kL1TileA, (n_bi + kL1TileB - 1) / kL1TileB);
  const uint32_t *ma, *mb;
  l1_masks(xa, yb, n_ai, n_bi, dim, grid, masks, &ma, &mb, s);
  l1_round_kernel<uint8_t, false><<<grid, 256, 0, s>>>(xa, yb, n_ai, n_bi, dim, 0.5, nullptr, 0, status, ma, mb);
  return cudaGetLastError();
}

__global__ void transpose_f64_kernel(const double* __restrict__ in, int n, int dim, double* __restrict__ out) {
  __shared__ double tile[32][33];
  const int i0 = blockIdx.x * 32, p0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, p = p0 + threadIdx.x;
    if (i < n && p < dim) tile[r][threadIdx.x] = in[(size_t)i * dim + p];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int p = p0 + r, i = i0 + threadIdx.x;
    if (i < n && p < dim) out[(size_t)p * n + i] = tile[threadIdx.x][r];
  }
}

cudaError_t launch_transpose_f64(const double* in, int n, int dim, double* out, cudaStream_t s) {
  transpose_f64_kernel<<<dim3((n + 31) / 32, (dim + 31) / 32), dim3(32, 8), 0, s>>>(in, n, dim, out);
  return cudaGetLastError();
}

cudaError_t launch_l1_matched_cost(const double* xa, const double* yb, int dim, const int32_t* match, int n,
                                   bool self_is_a, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  l1_matched_cost_kernel<<<(n + 127) / 128, 128, 0, s>>>(xa, yb, dim, match, n, self_is_a ? 1 : 0, out);
  return cudaGetLastError();
}

cudaError_t launch_points_matched_cost(const double* xa, const double* yb, const int32_t* match, int n,
                                       double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  points_matched_cost_kernel<<<(n + 255) / 256, 256, 0, s>>>(xa, yb, match, n, out);
  return cudaGetLastError();
}

cudaError_t launch_dense_matched_cost(const double* cost, int n_b, const int32_t* match, int n, double* out,
                                      cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  dense_matched_cost_kernel<<<(n + 255) / 256, 256, 0, s>>>(cost, n_b, match, n, out);
  return cudaGetLastError();
}

cudaError_t launch_k_to_kT(const int32_t* k, int n_a, int n_b, void* kT, int lda, int width,
                           cudaStream_t s) {
  dim3 block(32, 8), grid((lda + 31) / 32, (n_b + 31) / 32);
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    k_to_kT_kernel<T><<<grid, block, 0, s>>>(k, n_a, n_b, static_cast<T*>(kT), lda);
    return 0;
  });
  return cudaGetLastError();
}

cudaError_t launch_export_k(const void* kT, int n_ai, int n_bi, int lda, int width, bool swapped,
                            int32_t* k_out, cudaStream_t s) {
  with_width(width, [&](auto tag) {
    using T = decltype(tag);
    export_k_kernel<T><<<1184, 256, 0, s>>>(static_cast<const T*>(kT), n_ai, n_bi, lda, swapped, k_out);
    return 0;
  });
  return cudaGetLastError();
}

}  // namespace otprg
