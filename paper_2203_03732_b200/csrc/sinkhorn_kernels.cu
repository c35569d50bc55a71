// sinkhorn_kernels.cu — the entropic Sinkhorn baseline on the device
// (reference src/sinkhorn.cpp:69-151), FP64 throughout.
//
// The reference is a comparison point (plain kernel scaling, no log domain).
// Its work per iteration is two passes over the dense n_a x n_b kernel
// K = exp(-c/reg): row sums K v (for u and for the row-marginal violation)
// and column sums K^T u.  Here the violation pass of iteration i doubles as
// the u-update pass of iteration i+1 (same product K v_i), so an iteration
// is two HBM passes over K:
//   row pass    one warp per row, lanes stride the row (coalesced 8-byte
//               loads), shuffle-tree sum; fused |u s - mu| and mu / s;
//   column pass 256-column x 64-row tiles, one thread per column summing its
//               rows sequentially (coalesced across the warp), then the tile
//               partials summed in tile order.
// All reductions have a fixed order, so results are deterministic; they are
// not the reference's sequential sums bit for bit (nor is CUDA's exp glibc's),
// so parity is to a stated floating-point tolerance (tests/test_gpu_sinkhorn.py).
#include <cmath>

#include "device_common.cuh"
#include "kernels.h"

namespace otprg {

namespace {

constexpr int kColTile = 256;  // columns per column-pass block
constexpr int kRowTile = 64;   // rows per column-pass block

__global__ void sk_build_kernel(const double* __restrict__ cost, size_t total, int n_b, double reg,
                                double* __restrict__ K, int* __restrict__ row_ok,
                                int* __restrict__ col_ok, int* __restrict__ bad_cost) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const double c = cost[i];
    if (!(c >= 0.0 && c <= 1.0)) *bad_cost = 1;  // OTInstance::validate (ot.cpp:80-84)
    const double k = exp(__ddiv_rn(-c, reg));  // std::exp(-c / reg)  (sinkhorn.cpp:79-82)
    K[i] = k;
    if (k > 0.0) {
      row_ok[i / n_b] = 1;
      col_ok[i % n_b] = 1;
    }
  }
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(kFull, s, o));
  return s;
}

// s[a] = sum_b K[a][b] * v[b] (optionally times the row scale of P), and
//   term[a] = |u[a] s - mu[a]|, u_next[a] = mu[a] / s with error bits
//   (1: s not positive/finite, 2: u_next not finite), as sinkhorn.cpp:110-118.
__global__ void __launch_bounds__(256) sk_row_kernel(const double* __restrict__ K, int n_a, int n_b,
                                                     const double* __restrict__ u,
                                                     const double* __restrict__ v,
                                                     const double* __restrict__ mu,
                                                     double* __restrict__ term,
                                                     double* __restrict__ u_next, int* err) {
  const int lane = threadIdx.x & 31;
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n_a) return;
  const double* row = K + (size_t)a * n_b;
  double s = 0.0;
  for (int b = lane; b < n_b; b += 32) s = __dadd_rn(s, __dmul_rn(row[b], v[b]));
  s = warp_sum(s);
  if (lane == 0) {
    if (term) term[a] = fabs(__dsub_rn(__dmul_rn(u[a], s), mu[a]));
    int e = 0;
    if (!(s > 0.0) || !isfinite(s)) e |= 1;
    const double un = __ddiv_rn(mu[a], s);
    if (!isfinite(un)) e |= 2;
    u_next[a] = un;
    if (e) atomicOr(err, e);
  }
}

// Column pass, stage 1: partial[tile_row][b] = sum over the tile's rows of
// K[a][b] * w[a] (* P scales when `plan`).
__global__ void __launch_bounds__(kColTile) sk_col_partial_kernel(const double* __restrict__ K, int n_a,
                                                                  int n_b, const double* __restrict__ w,
                                                                  double* __restrict__ partial) {
  const int b = blockIdx.x * kColTile + threadIdx.x;
  const int a0 = blockIdx.y * kRowTile;
  if (b >= n_b) return;
  const int a1 = min(n_a, a0 + kRowTile);
  double s = 0.0;
#pragma unroll 8
  for (int a = a0; a < a1; ++a) s = __dadd_rn(s, __dmul_rn(K[(size_t)a * n_b + b], w[a]));
  partial[(size_t)blockIdx.y * n_b + b] = s;
}

// Column pass, stage 2: ktu[b] = partials in tile order; v[b] = nu[b] / ktu
// with error bits 4 / 8 (sinkhorn.cpp:120-128).
__global__ void sk_col_final_kernel(const double* __restrict__ partial, int tiles, int n_b,
                                    const double* __restrict__ nu, double* __restrict__ v, int* err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_b) return;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s = __dadd_rn(s, partial[(size_t)t * n_b + b]);
  if (!nu) {  // plain column sums (round_to_marginals)
    v[b] = s;
    return;
  }
  int e = 0;
  if (!(s > 0.0) || !isfinite(s)) e |= 4;
  const double vn = __ddiv_rn(nu[b], s);
  if (!isfinite(vn)) e |= 8;
  v[b] = vn;
  if (e) atomicOr(err, e);
}

// Deterministic sum of x[0..n) (one block): contiguous segments, then a tree.
__global__ void __launch_bounds__(1024) sk_sum_kernel(const double* __restrict__ x, int n, double* out) {
  __shared__ double sh[1024];
  const int t = threadIdx.x, nt = blockDim.x;
  const int chunk = (n + nt - 1) / nt;
  const int lo = min(n, t * chunk), hi = min(n, lo + chunk);
  double s = 0.0;
  for (int i = lo; i < hi; ++i) s = __dadd_rn(s, x[i]);
  sh[t] = s;
  __syncthreads();
  for (int o = nt / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] = __dadd_rn(sh[t], sh[t + o]);
    __syncthreads();
  }
  if (t == 0) *out = sh[0];
}

// Plan P(a,b) = u[a] * K(a,b) * v[b] (sinkhorn.cpp:144-146), then the row /
// column scales of round_to_marginals (:12-36) when given (only < 1 applied).
__global__ void sk_plan_kernel(const double* __restrict__ K, size_t total, int n_b,
                               const double* __restrict__ u, const double* __restrict__ v,
                               const double* __restrict__ rs, const double* __restrict__ cs,
                               double* __restrict__ P) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int a = (int)(i / n_b), b = (int)(i % n_b);
    double p = __dmul_rn(__dmul_rn(u[a], K[i]), v[b]);
    if (rs && rs[a] < 1.0) p = __dmul_rn(p, rs[a]);
    if (cs && cs[b] < 1.0) p = __dmul_rn(p, cs[b]);
    P[i] = p;
  }
}

// Row sums of P (warp per row) and the row scale mu/row when row > mu > 0 side.
__global__ void __launch_bounds__(256) sk_prow_kernel(const double* __restrict__ P, int n_a, int n_b,
                                                      const double* __restrict__ mu,
                                                      double* __restrict__ row,
                                                      double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n_a) return;
  const double* r = P + (size_t)a * n_b;
  double s = 0.0;
  for (int b = lane; b < n_b; b += 32) s = __dadd_rn(s, r[b]);
  s = warp_sum(s);
  if (lane == 0) {
    row[a] = s;
    if (scale) scale[a] = (s > mu[a] && s > 0.0) ? __ddiv_rn(mu[a], s) : 1.0;
  }
}

__global__ void sk_ones_kernel(double* w, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = 1.0;
}

__global__ void sk_colscale_kernel(const double* __restrict__ col, const double* __restrict__ nu,
                                   int n_b, double* __restrict__ scale) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n_b) scale[b] = (col[b] > nu[b] && col[b] > 0.0) ? __ddiv_rn(nu[b], col[b]) : 1.0;
}

// P[a][b] += add for the greedy fix-up entries (sinkhorn.cpp:52-62).
__global__ void sk_adds_kernel(double* __restrict__ P, int n_b, const int2* __restrict__ ab,
                               const double* __restrict__ add, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) P[(size_t)ab[i].x * n_b + ab[i].y] = __dadd_rn(P[(size_t)ab[i].x * n_b + ab[i].y], add[i]);
}

// Per row: positive entries and their cost contribution (row-ordered, warp tree).
__global__ void __launch_bounds__(256) sk_rowcost_kernel(const double* __restrict__ P,
                                                         const double* __restrict__ cost, int n_a,
                                                         int n_b, double* __restrict__ rcost,
                                                         long long* __restrict__ rcnt) {
  const int lane = threadIdx.x & 31;
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n_a) return;
  const double* r = P + (size_t)a * n_b;
  const double* c = cost + (size_t)a * n_b;
  double s = 0.0;
  int cnt = 0;
  for (int b = lane; b < n_b; b += 32) {
    const double p = r[b];
    if (p > 0.0) {
      s = __dadd_rn(s, __dmul_rn(p, c[b]));
      ++cnt;
    }
  }
  s = warp_sum(s);
  cnt = __reduce_add_sync(kFull, cnt);
  if (lane == 0) {
    rcost[a] = s;
    rcnt[a] = cnt;
  }
}

// Plan entries (row-major, p > 0) at offsets[a] (warp per row, ordered).
__global__ void __launch_bounds__(256) sk_entries_kernel(const double* __restrict__ P, int n_a, int n_b,
                                                         const long long* __restrict__ offs,
                                                         int32_t* __restrict__ ea,
                                                         int32_t* __restrict__ eb,
                                                         double* __restrict__ em) {
  const int lane = threadIdx.x & 31;
  const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (a >= n_a) return;
  const double* r = P + (size_t)a * n_b;
  long long pos = offs[a];
  for (int b0 = 0; b0 < n_b; b0 += 32) {
    const int b = b0 + lane;
    const double p = b < n_b ? r[b] : 0.0;
    const unsigned m = __ballot_sync(kFull, p > 0.0);
    if (p > 0.0) {
      const long long i = pos + __popc(m & ((1u << lane) - 1u));
      ea[i] = a;
      eb[i] = b;
      em[i] = p;
    }
    pos += __popc(m);
  }
}

}  // namespace

cudaError_t sk_build(const double* cost, int n_a, int n_b, double reg, double* K, int* row_ok,
                     int* col_ok, int* bad_cost, cudaStream_t s) {
  cudaMemsetAsync(row_ok, 0, n_a * sizeof(int), s);
  cudaMemsetAsync(col_ok, 0, n_b * sizeof(int), s);
  sk_build_kernel<<<148 * 8, 256, 0, s>>>(cost, (size_t)n_a * n_b, n_b, reg, K, row_ok, col_ok,
                                          bad_cost);
  return cudaGetLastError();
}

cudaError_t sk_row(const double* K, int n_a, int n_b, const double* u, const double* v,
                   const double* mu, double* term, double* u_next, int* err, cudaStream_t s) {
  sk_row_kernel<<<(n_a * 32 + 255) / 256, 256, 0, s>>>(K, n_a, n_b, u, v, mu, term, u_next, err);
  return cudaGetLastError();
}

cudaError_t sk_col(const double* K, int n_a, int n_b, const double* w, const double* nu, double* v,
                   double* partial, int* err, cudaStream_t s) {
  const int tiles = (n_a + kRowTile - 1) / kRowTile;
  sk_col_partial_kernel<<<dim3((n_b + kColTile - 1) / kColTile, tiles), kColTile, 0, s>>>(K, n_a, n_b, w,
                                                                                        partial);
  sk_col_final_kernel<<<(n_b + 255) / 256, 256, 0, s>>>(partial, tiles, n_b, nu, v, err);
  return cudaGetLastError();
}

size_t sk_partial_elems(int n_a, int n_b) { return (size_t)((n_a + kRowTile - 1) / kRowTile) * n_b; }

cudaError_t sk_sum(const double* x, int n, double* out, cudaStream_t s) {
  sk_sum_kernel<<<1, 1024, 0, s>>>(x, n, out);
  return cudaGetLastError();
}

cudaError_t sk_plan(const double* K, int n_a, int n_b, const double* u, const double* v,
                    const double* rs, const double* cs, double* P, cudaStream_t s) {
  sk_plan_kernel<<<148 * 8, 256, 0, s>>>(K, (size_t)n_a * n_b, n_b, u, v, rs, cs, P);
  return cudaGetLastError();
}

cudaError_t sk_prow(const double* P, int n_a, int n_b, const double* mu, double* row, double* scale,
                    cudaStream_t s) {
  sk_prow_kernel<<<(n_a * 32 + 255) / 256, 256, 0, s>>>(P, n_a, n_b, mu, row, scale);
  return cudaGetLastError();
}

// Column sums of P (weights 1) into col (through the partial buffer).
cudaError_t sk_pcol(const double* P, int n_a, int n_b, double* ones_a, double* partial, double* col,
                    cudaStream_t s) {
  sk_ones_kernel<<<(n_a + 255) / 256, 256, 0, s>>>(ones_a, n_a);
  const int tiles = (n_a + kRowTile - 1) / kRowTile;
  sk_col_partial_kernel<<<dim3((n_b + kColTile - 1) / kColTile, tiles), kColTile, 0, s>>>(P, n_a, n_b,
                                                                                        ones_a, partial);
  // the final stage without the division: reuse sum order, write the sums
  sk_col_final_kernel<<<(n_b + 255) / 256, 256, 0, s>>>(partial, tiles, n_b, nullptr, col, nullptr);
  return cudaGetLastError();
}

cudaError_t sk_colscale(const double* col, const double* nu, int n_b, double* scale, cudaStream_t s) {
  sk_colscale_kernel<<<(n_b + 255) / 256, 256, 0, s>>>(col, nu, n_b, scale);
  return cudaGetLastError();
}

cudaError_t sk_adds(double* P, int n_b, const int2* ab, const double* add, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  sk_adds_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, n_b, ab, add, n);
  return cudaGetLastError();
}

cudaError_t sk_rowcost(const double* P, const double* cost, int n_a, int n_b, double* rcost,
                       long long* rcnt, cudaStream_t s) {
  sk_rowcost_kernel<<<(n_a * 32 + 255) / 256, 256, 0, s>>>(P, cost, n_a, n_b, rcost, rcnt);
  return cudaGetLastError();
}

cudaError_t sk_entries(const double* P, int n_a, int n_b, const long long* offs, int32_t* ea,
                       int32_t* eb, double* em, cudaStream_t s) {
  sk_entries_kernel<<<(n_a * 32 + 255) / 256, 256, 0, s>>>(P, n_a, n_b, offs, ea, eb, em);
  return cudaGetLastError();
}

}  // namespace otprg
