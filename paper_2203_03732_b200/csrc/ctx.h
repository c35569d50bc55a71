// ctx.h — the otprg_ctx behind the C ABI (internal to libotprg.so).
#pragma once
#include <cmath>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/otprg.h"

namespace otprg {

// Grow-only device buffer.
struct DevBuf {  // owning, move-free device buffer (freed with its context)
  void* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// scaled_floor, core.cpp:26-32 (host copy).
inline int64_t host_scaled_floor(double c, double eps) {
  auto k = static_cast<int64_t>(std::floor(c / eps));
  while (static_cast<double>(k + 1) * eps <= c) ++k;
  while (k > 0 && static_cast<double>(k) * eps > c) --k;
  return k;
}

}  // namespace otprg

struct otprg_ctx;
namespace otprg {
// Large H2D from caller memory that may be pageable (h2d.cpp).
cudaError_t h2d_large(otprg_ctx* ctx, void* dst, const void* src, size_t bytes);
void release_bounce(otprg_ctx* ctx);
}  // namespace otprg

struct otprg_ctx {
  using DevBuf = otprg::DevBuf;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;  // created by otprg_create (stream may be the caller's)
  cudaEvent_t ev[8] = {};
  int num_sms = 0;
  std::string err;

  // prepared assignment problem
  bool prepared = false;
  int32_t n_a = 0, n_b = 0;  // original orientation
  int32_t ia = 0, ib = 0;    // internal: ia >= ib
  bool swapped = false;
  int width = 1, lda = 0;
  double eps = 0.0;
  int32_t unit_floor = 0, unit_ceil = 0;
  int cost_kind = 0;
  const double* host_cost = nullptr;  // caller buffer (DENSE); valid until next prepare
  bool stage_holds_cost = false;      // stage = the prepared dense f64 matrix (caller orientation)
  std::vector<double> pts_a, pts_b;   // original orientation (POINTS2D)
  std::vector<uint8_t> img_a, img_b;  // original orientation (L1_U8)
  int img_dim = 0;
  double build_ms = 0.0;
  int build_launches = 0;

  DevBuf kT, t, yb, ma, mb, holder, rowmin, lmeta, lent, lists, mps, fc, ctl, fa, fb;
  DevBuf stage, pts, flush;
  DevBuf l1_mask;  // K3 tile pixel-support masks
  DevBuf k2_fix;   // K2 rows deferred to the exact fix-up pass
  DevBuf l1_otf_mask;  // on-the-fly L1: demand group / supply image pixel-support masks
  // exact threshold table of the 2-D point cost for eps = thr_eps (K2 and the
  // on-the-fly scans; otprg_points_threshold_table), cached across prepares
  DevBuf thr_dev, range_first;
  std::vector<double> thr_host;
  double thr_eps = -1.0;
  int thr_n = 0;
  double pts_absmax = 1.0;  // largest |coordinate| of the prepared point sets (K2's error bound)
  void* hpin = nullptr;  // pinned D2H staging
  size_t hpin_n = 0;
  cudaEvent_t timer[2] = {};
  int64_t fc_cap = 0;
  int loop_grid = 0;
  bool smem_t = true;
  bool begun = false, completed = false;
  DevBuf trace;            // device timeline, 8 u64 per phase (see solve_kernels.cu)
  uint32_t trace_cap = 0;  // 0 = tracing off

  // A-row-sharded mode (shard_kernels.cu, shard_host.cpp): this shard's slab [sh_lo, sh_hi)
  bool sharded = false;
  int sh_n_shards = 1, sh_shard = 0, sh_lo = 0, sh_hi = 0, sh_K = 16, sh_cap = 0;
  int sh_grid = 0, sh_da_grid = 0;  // resident-sized grids of the scan / DA kernels
  uint64_t sh_gen = 0;              // bumped by every shard prepare (invalidates resident plans)
  // host-driven protocol: the round state last read back from the device
  bool sh_have = false;
  int sh_n = 0, sh_parked = 0, sh_done = 0;
  uint32_t sh_epoch = 0;            // exchange epochs used so far (flags only grow)
  DevBuf sh_bounds, sh_pos, sh_park[2], sh_list, sh_seg;
  bool sh_otf = false;  // OTPRG_FLAG_ON_THE_FLY: no kT slab, threshold-table scans
  bool sh_otf_tiled = true;
  int sh_thr_n = 0;
  size_t sh_l1_xt = 0;  // on-the-fly L1: byte offset of the transposed demand pixels in pts
  std::shared_ptr<void> sh_plan;    // resident loop (graphs, exchange blocks, peers): shard_host.cpp
  // multi-device context (otprg_create_multi): one shard context per device
  std::vector<otprg_ctx*> multi;
  int multi_K = 16;
  bool multi_prepared = false;

  // invariant suite / workset export (verify_kernels.cu)
  DevBuf v_out, v_k, v_ya, v_yb, v_ma, v_mb, adm_cnt, adm_off, adm_list;

  // copy mode (copy_kernels.cu): groups, per-phase order, host-side stats
  bool groups_mode = false, g_done = false, g_full = false;
  int g_ndg = 0, g_nsg = 0;
  uint32_t g_phase = 0;
  int64_t g_sum_ni = 0;
  std::vector<int64_t> g_fc;
  DevBuf g_d, g_s, g_keys, g_keys2, g_vals, g_pi, g_rank, g_tmp, g_gmax, g_cnt;

  // pinned bounce buffers for large copies from pageable host memory (h2d.cpp)
  void* bounce[2] = {nullptr, nullptr};
  cudaEvent_t bounce_ev[2] = {nullptr, nullptr};

  // Sinkhorn baseline (ot_host.cpp / sinkhorn_kernels.cu)
  DevBuf sk_K, sk_P, sk_vec, sk_part, sk_int;

  // optimal transport (ot_host.cpp): per-phase scan inputs / outputs
  DevBuf ot_t, ot_req, ot_out;
  DevBuf ot_dev[48];  // the OT cluster state and phase buffers on the device (ot_host.cpp)
  void* ot_hpin = nullptr;
  std::shared_ptr<void> ot_state;  // flat ClusterState of the last copy/cluster solve (ot_host.cpp)
  size_t ot_hpin_n = 0;
};
