// otprg_capi.cpp — host side of the C ABI declared in include/otprg.h.
//
// Validation, storage choice, device buffers and the launch sequence of the
// assignment path:
//   H2D -> cost build/rounding (K1 dense / K2 points) -> init_state ->
//   phase loop (phase 1 as its own launch, then the rest) -> completion ->
//   D2H -> matching cost on the host.
// Mirrors otpr::solve_assignment (src/assignment.cpp:368-400) and
// otpr::scale_round_costs (src/core.cpp:34-53).  Built with
// -ffp-contract=off so the host-side cost sums match the reference bits.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/otprg.h"
#include "kernels.h"

using otprg::Ctl;

#include "ctx.h"
#include "capi_internal.h"

using otprg::DevBuf;
using otprg::host_scaled_floor;

namespace otprg_capi {

int fail(otprg_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(otprg_ctx* ctx, cudaError_t e, const char* what) {
  return fail(ctx, OTPRG_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}


// Validation of solve_assignment (assignment.cpp:370-372) and
// scale_round_costs (core.cpp:35-47) that does not need the cost values.
int validate_problem(otprg_ctx* ctx, const otprg_problem* p) {
  if (!p) return fail(ctx, OTPRG_PARAMETER, "null problem");
  if (p->n_a < 1 || p->n_b < 1)
    return fail(ctx, OTPRG_PARAMETER, "instance needs at least one vertex per side");
  if (!(p->eps > 0.0 && p->eps < 1.0))
    return fail(ctx, OTPRG_PARAMETER, "eps must lie in (0, 1), got " + std::to_string(p->eps));
  const int64_t uf = host_scaled_floor(1.0, p->eps);
  if (uf + 4 > std::numeric_limits<int32_t>::max())
    return fail(ctx, OTPRG_PARAMETER, "eps too small: 1/eps overflows the cost unit type");
  switch (p->cost_kind) {
    case OTPRG_COST_DENSE_F64:
      if (!p->cost) return fail(ctx, OTPRG_PARAMETER, "dense cost pointer is null");
      break;
    case OTPRG_COST_POINTS2D:
      if (!p->pts_a || !p->pts_b) return fail(ctx, OTPRG_PARAMETER, "point pointers are null");
      break;
    case OTPRG_COST_L1_U8:
      if (!p->img_a || !p->img_b || p->dim < 1)
        return fail(ctx, OTPRG_PARAMETER, "image pointers are null or dim < 1");
      break;
    default:
      return fail(ctx, OTPRG_PARAMETER, "unsupported cost kind " + std::to_string(p->cost_kind));
  }
  return OTPRG_OK;
}

// Largest d2 whose point cost RN(RN(sqrt(d2)) / sqrt(2)) is <= 1 (bisection
// over the bit patterns; the cost is monotone in d2).
double points_d2_max() {
  static const double v = [] {
    const double sqrt2 = std::sqrt(2.0);
    auto bits = [](double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; };
    auto from = [](uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; };
    uint64_t lo = bits(2.0), hi = bits(8.0);  // cost(lo) <= 1 < cost(hi)
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (std::sqrt(from(mid)) / sqrt2 <= 1.0) lo = mid;
      else hi = mid;
    }
    return from(lo);
  }();
  return v;
}

// AssignmentInstance::validate (core.cpp:15-21) for a point instance: every
// cost sqrt(dx*dx+dy*dy)/sqrt(2) must lie in [0, 1].  The bounding box of both
// sets bounds every pair's d2 (RN arithmetic is monotone), which settles it
// for any points inside the unit square; otherwise a device pass finds the
// first violating (a, b) in row-major order, reported with the reference's
// message.  dpa_orig / dpb_orig: device copies of the original A / B points.
int check_points_range(otprg_ctx* ctx, const otprg_problem* p, const double* dpa_orig,
                       const double* dpb_orig) {
  double lo[2] = {INFINITY, INFINITY}, hi[2] = {-INFINITY, -INFINITY};
  bool nan = false;
  for (int side = 0; side < 2; ++side) {
    const double* q = side ? p->pts_b : p->pts_a;
    const int64_t n = side ? p->n_b : p->n_a;
    for (int64_t i = 0; i < 2 * n; ++i) {
      const double x = q[i];
      if (x != x) nan = true;
      lo[i & 1] = std::min(lo[i & 1], x);
      hi[i & 1] = std::max(hi[i & 1], x);
    }
  }
  ctx->pts_absmax = std::max(std::max(std::fabs(lo[0]), std::fabs(hi[0])), std::max(std::fabs(lo[1]), std::fabs(hi[1])));
  if (!nan) {
    const double dx = hi[0] - lo[0], dy = hi[1] - lo[1];
    if (dx * dx + dy * dy <= points_d2_max()) return OTPRG_OK;
  }
  CK(ctx->range_first.ensure(8), "alloc range flag");
  CK(cudaMemsetAsync(ctx->range_first.p, 0xff, 8, ctx->stream), "memset");
  CK(otprg::launch_points_range(dpa_orig, dpb_orig, p->n_a, p->n_b, points_d2_max(),
                                ctx->range_first.as<unsigned long long>(), ctx->stream),
     "range check launch");
  unsigned long long first = 0;
  CK(cudaMemcpyAsync(&first, ctx->range_first.p, 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  CK(cudaStreamSynchronize(ctx->stream), "range check");
  if (first == ~0ull) return OTPRG_OK;
  const int64_t a = static_cast<int64_t>(first / p->n_b), b = static_cast<int64_t>(first % p->n_b);
  const double dx = p->pts_a[2 * a] - p->pts_b[2 * b], dy = p->pts_a[2 * a + 1] - p->pts_b[2 * b + 1];
  const double c = std::sqrt(dx * dx + dy * dy) / std::sqrt(2.0);
  return fail(ctx, OTPRG_PARAMETER, "cost entry outside [0,1] at (" + std::to_string(a) + "," +
                                        std::to_string(b) + "): " + std::to_string(c));
}

// The exact threshold table for eps on the device (cached per eps).  Returns
// its length, 0 when it is too large for the shared-memory kernels.
int points_table(otprg_ctx* ctx, double eps, int* n_out) {
  *n_out = 0;
  const int32_t n = otprg_points_threshold_table(eps, nullptr, 0);
  if (n < 2 || n > 8192) return OTPRG_OK;
  if (ctx->thr_eps != eps || ctx->thr_n != n) {
    ctx->thr_host.assign(n, 0.0);
    otprg_points_threshold_table(eps, ctx->thr_host.data(), n);
    CK(ctx->thr_dev.ensure(n * sizeof(double)), "alloc threshold table");
    CK(cudaMemcpyAsync(ctx->thr_dev.p, ctx->thr_host.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream),
       "H2D threshold table");
    ctx->thr_eps = eps;
    ctx->thr_n = n;
  }
  *n_out = n;
  return OTPRG_OK;
}

int do_prepare(otprg_ctx* ctx, const otprg_problem* p) {
  int st = validate_problem(ctx, p);
  if (st) return st;
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->prepared = false;
  ctx->sharded = false;  // (a shard_prepare on this context is superseded)
  ctx->n_a = p->n_a;
  ctx->n_b = p->n_b;
  ctx->swapped = p->n_b > p->n_a;  // assignment.cpp:385-399
  ctx->ia = ctx->swapped ? p->n_b : p->n_a;
  ctx->ib = ctx->swapped ? p->n_a : p->n_b;
  ctx->eps = p->eps;
  ctx->cost_kind = p->cost_kind;
  const int64_t uf = host_scaled_floor(1.0, p->eps);
  ctx->unit_floor = static_cast<int32_t>(uf);
  ctx->unit_ceil = static_cast<int32_t>(static_cast<double>(uf) * p->eps == 1.0 ? uf : uf + 1);

  // Storage: |Y| <= unit_ceil + 2 (core.hpp:94-95) must stay below the
  // saturation value of the packed k + t sums.
  const int64_t need = static_cast<int64_t>(ctx->unit_ceil) + 2;
  const int width = otprg::storage_width(need, p->storage);
  if (width < 0)
    return fail(ctx, OTPRG_PARAMETER,
                "eps too small for the device cost storage (ceil(1/eps)+2 = " +
                    std::to_string(need) + ")");
  ctx->width = width;
  const int align = 512 / width;
  ctx->lda = (ctx->ia + align - 1) / align * align;

  const size_t ia = ctx->ia, ib = ctx->ib, lda = ctx->lda;
  CK(ctx->kT.ensure(ib * lda * width), "alloc kT");
  CK(ctx->t.ensure(lda * width), "alloc t");
  CK(ctx->yb.ensure(ib * 4), "alloc yb");
  CK(ctx->ma.ensure(ia * 4), "alloc match_a");
  CK(ctx->mb.ensure(ib * 4), "alloc match_b");
  CK(ctx->holder.ensure(2 * ia * 8), "alloc holder");
  CK(ctx->rowmin.ensure(ib * width), "alloc rowmin");
  CK(ctx->lmeta.ensure(ib * 16), "alloc low-set meta");
  CK(ctx->lent.ensure(ib * 8 * otprg::kLowCap), "alloc low-set entries");
  CK(ctx->lists.ensure(3 * ib * 4), "alloc lists");
  CK(ctx->mps.ensure(3 * ib * 8), "alloc mp lists");
  CK(ctx->fa.ensure(ia * 4), "alloc scratch");
  CK(ctx->fb.ensure(ib * 4), "alloc scratch");
  CK(ctx->ctl.ensure(sizeof(Ctl)), "alloc ctl");
  const double capd = std::ceil((1.0 + 2.0 * p->eps) / (p->eps * p->eps)) + 8.0;
  ctx->fc_cap = static_cast<int64_t>(std::min(capd + 1.0, double(OTPRG_MAX_PHASES)));
  CK(ctx->fc.ensure(ctx->fc_cap * 8), "alloc free_counts");
  ctx->smem_t = otprg::smem_t_fits(width, ctx->lda);
  ctx->loop_grid = otprg::phase_loop_grid(width, ctx->smem_t, ctx->lda, ctx->num_sms);
  if (ctx->loop_grid <= 0) return fail(ctx, OTPRG_DEVICE, "phase loop kernel cannot be resident");

  CK(cudaEventRecord(ctx->ev[4], ctx->stream), "event");
  ctx->build_launches = 0;
  if (p->cost_kind == OTPRG_COST_DENSE_F64) {
    const size_t bytes = static_cast<size_t>(p->n_a) * p->n_b * sizeof(double);
    ctx->stage_holds_cost = false;
    CK(ctx->stage.ensure(bytes), "alloc cost staging");
    CK(otprg::h2d_large(ctx, ctx->stage.p, p->cost, bytes), "H2D cost");
    ctx->stage_holds_cost = true;
    CK(cudaMemsetAsync(ctx->ctl.p, 0, sizeof(Ctl), ctx->stream), "memset");
    int* status = &ctx->ctl.as<Ctl>()->status;
    CK(otprg::launch_round_dense(ctx->stage.as<double>(), p->n_a, p->n_b, ctx->swapped, p->eps,
                                 ctx->kT.p, ctx->lda, width, status, ctx->stream),
       "round_dense launch");
    ctx->build_launches = 1;
    ctx->host_cost = p->cost;
  } else if (p->cost_kind == OTPRG_COST_L1_U8) {
    ctx->stage_holds_cost = false;
    // load_mnist_pair's cost (instances.cpp:114-142) from raw pixels
    const size_t dim = static_cast<size_t>(p->dim);
    const uint8_t* ia_img = ctx->swapped ? p->img_b : p->img_a;  // internal demand side
    const uint8_t* ib_img = ctx->swapped ? p->img_a : p->img_b;
    CK(ctx->pts.ensure((ia + ib) * dim * (sizeof(double) + 1)), "alloc images");
    double* xa = ctx->pts.as<double>();
    double* yb = xa + ia * dim;
    uint8_t* raw = reinterpret_cast<uint8_t*>(yb + ib * dim);
    CK(cudaMemcpyAsync(raw, ia_img, ia * dim, cudaMemcpyHostToDevice, ctx->stream), "H2D images");
    CK(cudaMemcpyAsync(raw + ia * dim, ib_img, ib * dim, cudaMemcpyHostToDevice, ctx->stream),
       "H2D images");
    CK(cudaMemsetAsync(ctx->ctl.p, 0, sizeof(Ctl), ctx->stream), "memset");
    int* status = &ctx->ctl.as<Ctl>()->status;
    CK(otprg::launch_l1_normalize(raw, static_cast<int>(ia + ib), p->dim, xa, status, ctx->stream),
       "l1 normalize launch");
    CK(ctx->l1_mask.ensure(otprg::l1_mask_bytes(ctx->ia, ctx->ib, ctx->lda, p->dim)), "alloc masks");
    CK(otprg::launch_l1_round(xa, yb, ctx->ia, ctx->ib, p->dim, p->eps, ctx->kT.p, ctx->lda, width,
                              status, ctx->stream, ctx->l1_mask.as<uint32_t>()),
       "l1 round launch");
    ctx->build_launches = 4;
    ctx->img_dim = p->dim;
    ctx->img_a.assign(p->img_a, p->img_a + dim * p->n_a);
    ctx->img_b.assign(p->img_b, p->img_b + dim * p->n_b);
  } else {
    ctx->stage_holds_cost = false;
    const double* pa = ctx->swapped ? p->pts_b : p->pts_a;  // internal demand points
    const double* pb = ctx->swapped ? p->pts_a : p->pts_b;
    CK(ctx->pts.ensure((ia + ib) * 2 * sizeof(double)), "alloc points");
    double* dpa = ctx->pts.as<double>();
    double* dpb = dpa + ia * 2;
    CK(cudaMemcpyAsync(dpa, pa, ia * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
       "H2D points");
    CK(cudaMemcpyAsync(dpb, pb, ib * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
       "H2D points");
    CK(cudaMemsetAsync(ctx->ctl.p, 0, sizeof(Ctl), ctx->stream), "memset");
    st = check_points_range(ctx, p, ctx->swapped ? dpb : dpa, ctx->swapped ? dpa : dpb);
    if (st) return st;
    int thr_n = 0;
    if ((st = points_table(ctx, p->eps, &thr_n))) return st;
    const size_t fix_bytes =
        otprg::round_points_fix_bytes(ctx->ia, ctx->ib, ctx->lda, width, p->eps, ctx->pts_absmax);
    CK(ctx->k2_fix.ensure(fix_bytes), "alloc K2 fix-up list");
    CK(otprg::launch_round_points2d(dpa, dpb, ctx->ia, ctx->ib, p->eps, std::sqrt(2.0),
                                    thr_n ? ctx->thr_dev.as<double>() : nullptr, thr_n, ctx->pts_absmax, ctx->kT.p,
                                    ctx->lda, width, ctx->k2_fix.p, fix_bytes, ctx->stream),
       "round_points launch");
    ctx->build_launches = thr_n ? 2 : 1;
    ctx->pts_a.assign(p->pts_a, p->pts_a + 2 * static_cast<size_t>(p->n_a));
    ctx->pts_b.assign(p->pts_b, p->pts_b + 2 * static_cast<size_t>(p->n_b));
  }
  CK(cudaEventRecord(ctx->ev[5], ctx->stream), "event");
  int dstatus = 0;
  CK(cudaMemcpyAsync(&dstatus, &ctx->ctl.as<Ctl>()->status, sizeof(int), cudaMemcpyDeviceToHost,
                     ctx->stream),
     "D2H status");
  CK(cudaStreamSynchronize(ctx->stream), "cost build");
  if (dstatus == OTPRG_PARAMETER) return fail(ctx, OTPRG_PARAMETER, "cost entry outside [0,1]");
  if (dstatus == OTPRG_INPUT) return fail(ctx, OTPRG_INPUT, "image has zero total intensity");
  if (dstatus) return fail(ctx, dstatus, "cost build failed");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]);
  ctx->build_ms = ms;
  ctx->prepared = true;
  return OTPRG_OK;
}

// L1/2 of two normalised images, ascending p (instances.cpp:116-126,134-141).
double l1_cost(const uint8_t* x, const uint8_t* y, int dim) {
  double tx = 0.0, ty = 0.0;
  for (int p = 0; p < dim; ++p) tx += x[p];
  for (int p = 0; p < dim; ++p) ty += y[p];
  double l1 = 0.0;
  for (int p = 0; p < dim; ++p)
    l1 += std::abs(static_cast<double>(x[p]) / tx - static_cast<double>(y[p]) / ty);
  return l1 / 2.0;
}

double pair_cost(const otprg_ctx* ctx, int32_t a, int32_t b) {
  if (ctx->cost_kind == OTPRG_COST_DENSE_F64)
    return ctx->host_cost[static_cast<size_t>(a) * ctx->n_b + b];
  if (ctx->cost_kind == OTPRG_COST_L1_U8)
    return l1_cost(ctx->img_a.data() + static_cast<size_t>(a) * ctx->img_dim,
                   ctx->img_b.data() + static_cast<size_t>(b) * ctx->img_dim, ctx->img_dim);
  // instances.cpp:70-75, same expression, non-fused (-ffp-contract=off)
  const double sqrt2 = std::sqrt(2.0);
  const double dx = ctx->pts_a[2 * static_cast<size_t>(a)] - ctx->pts_b[2 * static_cast<size_t>(b)];
  const double dy =
      ctx->pts_a[2 * static_cast<size_t>(a) + 1] - ctx->pts_b[2 * static_cast<size_t>(b) + 1];
  return std::sqrt(dx * dx + dy * dy) / sqrt2;
}

otprg::SolveArgs make_args(otprg_ctx* ctx) {
  otprg::SolveArgs A{};
  A.kT = ctx->kT.p;
  A.t = ctx->t.p;
  A.yb = ctx->yb.as<int32_t>();
  A.match_a = ctx->ma.as<int32_t>();
  A.match_b = ctx->mb.as<int32_t>();
  A.holder[0] = ctx->holder.as<unsigned long long>();
  A.holder[1] = A.holder[0] + ctx->ia;
  A.rowmin = ctx->rowmin.p;
  A.lmeta = ctx->lmeta.as<int4>();
  A.lent = ctx->lent.as<unsigned long long>();
  for (int r = 0; r < 3; ++r) {
    A.list[r] = ctx->lists.as<int32_t>() + static_cast<size_t>(r) * ctx->ib;
    A.mp[r] = ctx->mps.as<int2>() + static_cast<size_t>(r) * ctx->ib;
  }
  A.free_counts = ctx->fc.as<int64_t>();
  A.ctl = ctx->ctl.as<Ctl>();
  A.trace = ctx->trace_cap ? ctx->trace.as<unsigned long long>() : nullptr;
  A.trace_cap = ctx->trace_cap;
  A.pre_scanned = 1;  // do_begin always runs the phase-1 propose scan
  return A;
}

// init_state (assignment.cpp:54-60) + loop control block + the phase-1
// propose scan.  Events (optional): before init, after init, after the scan.
int do_begin(otprg_ctx* ctx, cudaEvent_t ev_init = nullptr, cudaEvent_t ev_scan0 = nullptr,
             cudaEvent_t ev_scan1 = nullptr) {
  if (!ctx->prepared) return fail(ctx, OTPRG_PARAMETER, "no prepared problem");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  Ctl h{};
  h.n_a = ctx->ia;
  h.n_b = ctx->ib;
  h.lda = ctx->lda;
  // (double)n_i <= eps * m  <=>  n_i <= floor(eps * m)   (assignment.cpp:324-331)
  const double threshold = ctx->eps * static_cast<double>(std::min(ctx->n_a, ctx->n_b));
  h.thresh = static_cast<int32_t>(std::floor(threshold));
  h.phase_cap = static_cast<int32_t>(ctx->fc_cap - 1);
  h.tmax = otprg::storage_tmax(ctx->width);
  h.cnt[0] = ctx->ib;  // phase 1 reads list 0 (all b)
  h.slots[0] = ctx->ib;
  h.prop_t0 = ~0ull;
  const otprg::SolveArgs A = make_args(ctx);
  CK(cudaMemcpyAsync(ctx->ctl.p, &h, sizeof(Ctl), cudaMemcpyHostToDevice, ctx->stream), "H2D ctl");
  if (ev_init) CK(cudaEventRecord(ev_init, ctx->stream), "event");
  CK(otprg::launch_init_state(A, ctx->ia, ctx->ib, ctx->lda, ctx->width, ctx->stream),
     "init launch");
  if (ev_scan0) CK(cudaEventRecord(ev_scan0, ctx->stream), "event");
  CK(otprg::launch_propose_stream(ctx->kT.p, ctx->lda, ctx->ib, ctx->width, A.lmeta, A.lent,
                                  ctx->rowmin.p, A.ctl, ctx->num_sms, ctx->stream),
     "propose scan launch");
  if (ev_scan1) CK(cudaEventRecord(ev_scan1, ctx->stream), "event");
  if (ctx->trace_cap)
    CK(cudaMemsetAsync(ctx->trace.p, 0, ctx->trace_cap * 8ull * otprg::kTraceSlots, ctx->stream), "trace reset");
  ctx->begun = true;
  ctx->completed = false;
  return OTPRG_OK;
}

int launch_loop(otprg_ctx* ctx, uint32_t max_phase) {
  otprg::SolveArgs A = make_args(ctx);
  A.max_phase = max_phase;
  CK(otprg::launch_phase_loop(A, ctx->width, ctx->smem_t, ctx->lda, ctx->loop_grid, ctx->stream),
     "phase loop launch");
  return OTPRG_OK;
}

int launch_finish(otprg_ctx* ctx) {
  CK(otprg::launch_complete(ctx->ma.as<int32_t>(), ctx->mb.as<int32_t>(), ctx->ia, ctx->ib,
                            ctx->fa.as<int32_t>(), ctx->fb.as<int32_t>(), ctx->stream),
     "complete launch");
  ctx->completed = true;
  return OTPRG_OK;
}

// Device status words (Ctl::status; details in Ctl::err[], see report()).
int check_status(otprg_ctx* ctx, const Ctl& h, bool need_done) {
  if (h.status == 0) {
    if (need_done && !h.done) return fail(ctx, OTPRG_DEVICE, "phase loop ended without termination");
    return OTPRG_OK;
  }
  std::string d;
  for (int i = 0; i < 6; ++i) d += (i ? "," : "") + std::to_string(h.err[i]);
  switch (h.status) {
    case 5:
      return fail(ctx, OTPRG_INVARIANT,
                  "phase count exceeded the proven bound; solver state is corrupt");
    case 6: return fail(ctx, OTPRG_DEVICE, "device grid barrier timeout (block " + d + ")");
    case 7: return fail(ctx, OTPRG_INVARIANT, "proposal conservation violated [phase,n,held,unmatched]=" + d);
    case 8: return fail(ctx, OTPRG_INVARIANT, "scan missed an admissible edge [phase,b,start,a,x,target]=" + d);
    case 9: return fail(ctx, OTPRG_INVARIANT, "scan returned an inadmissible edge [phase,b,start,a,k*1000+t,target]=" + d);
    case 10: return fail(ctx, OTPRG_INVARIANT, "state inconsistent after phase [phase,list,free,bad_b]=" + d);
    case 11: return fail(ctx, OTPRG_INVARIANT, "supply dual exceeded the device storage bound [phase,b,y]=" + d);
    case 12: return fail(ctx, OTPRG_INVARIANT, "demand dual exceeded the device storage bound [phase,a,t]=" + d);
    case 13: return fail(ctx, OTPRG_INVARIANT, "holder key from a later phase [phase,b,a,key_phase,key_b]=" + d);
    case 14: return fail(ctx, OTPRG_DEVICE, "tail loop entered above its team-size regime [phase,slots]=" + d);
    default: return fail(ctx, h.status, "device solve failed [" + d + "]");
  }
}

// Whether export_state evaluates the matched-pair costs on the device.
bool dev_pair_costs(const otprg_ctx* ctx) {
  return ctx->cost_kind == OTPRG_COST_L1_U8 || ctx->cost_kind == OTPRG_COST_POINTS2D ||
         (ctx->cost_kind == OTPRG_COST_DENSE_F64 && ctx->stage_holds_cost);
}

// Copies the current device state into the caller's result (caller
// orientation for the matching; internal orientation for the duals).
int export_state(otprg_ctx* ctx, otprg_result* r, Ctl* hout) {
  const int ia = ctx->ia, ib = ctx->ib;
  cudaStream_t s = ctx->stream;
  // One batch of async copies into pinned staging, one sync.
  const size_t o_ma = (sizeof(Ctl) + 255) / 256 * 256, o_mb = o_ma + ia * 4ull, o_yb = o_mb + ib * 4ull,
               o_t = o_yb + ib * 4ull, o_fc = (o_t + static_cast<size_t>(ia) * ctx->width + 7) & ~7ull;
  const int64_t fc_first = std::min<int64_t>(
      std::min<int64_t>(ctx->fc_cap, r->free_counts ? r->free_cap : 0), 65536);
  // Costs of the matched pairs are evaluated on the device (the reference's
  // arithmetic: L1 over K3's normalised pixels, the point formula, or a
  // gather from the dense matrix), one per original a; the host only sums.
  const bool l1 = ctx->cost_kind == OTPRG_COST_L1_U8;
  const bool dev_pc = dev_pair_costs(ctx);
  const size_t o_pc = o_fc + static_cast<size_t>(fc_first) * 8;
  const size_t need = o_pc + (dev_pc ? static_cast<size_t>(ctx->n_a) * 8 : 0);
  if (ctx->hpin_n < need) {
    if (ctx->hpin) cudaFreeHost(ctx->hpin);
    ctx->hpin = nullptr;
    ctx->hpin_n = 0;
    CK(cudaMallocHost(&ctx->hpin, need), "pinned staging");
    ctx->hpin_n = need;
  }
  char* hp = static_cast<char*>(ctx->hpin);
  CK(cudaMemcpyAsync(hp, ctx->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s), "D2H ctl");
  CK(cudaMemcpyAsync(hp + o_ma, ctx->ma.p, ia * 4ull, cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(hp + o_mb, ctx->mb.p, ib * 4ull, cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(hp + o_yb, ctx->yb.p, ib * 4ull, cudaMemcpyDeviceToHost, s), "D2H");
  CK(cudaMemcpyAsync(hp + o_t, ctx->t.p, static_cast<size_t>(ia) * ctx->width,
                     cudaMemcpyDeviceToHost, s), "D2H");
  if (fc_first > 0)
    CK(cudaMemcpyAsync(hp + o_fc, ctx->fc.p, fc_first * 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (dev_pc) {
    CK(ctx->v_ya.ensure(static_cast<size_t>(ctx->n_a) * 8), "alloc pair costs");
    // original a = internal a (unswapped, partner match_a) or internal b (swapped, partner match_b)
    const int32_t* m_orig = ctx->swapped ? ctx->mb.as<int32_t>() : ctx->ma.as<int32_t>();
    if (l1) {
      const size_t dim = ctx->img_dim;
      const double* xa = ctx->pts.as<double>();
      const double* yb = xa + static_cast<size_t>(ctx->ia) * dim;
      CK(otprg::launch_l1_matched_cost(xa, yb, ctx->img_dim, m_orig, ctx->n_a, !ctx->swapped,
                                       ctx->v_ya.as<double>(), s),
         "pair cost launch");
    } else if (ctx->cost_kind == OTPRG_COST_POINTS2D) {
      const double* dpa = ctx->pts.as<double>();  // internal demand points, then supply points
      const double* dpb = dpa + static_cast<size_t>(ia) * 2;
      CK(otprg::launch_points_matched_cost(ctx->swapped ? dpb : dpa, ctx->swapped ? dpa : dpb, m_orig, ctx->n_a,
                                           ctx->v_ya.as<double>(), s),
         "pair cost launch");
    } else {
      CK(otprg::launch_dense_matched_cost(ctx->stage.as<double>(), ctx->n_b, m_orig, ctx->n_a,
                                          ctx->v_ya.as<double>(), s),
         "pair cost launch");
    }
    CK(cudaMemcpyAsync(hp + o_pc, ctx->v_ya.p, static_cast<size_t>(ctx->n_a) * 8, cudaMemcpyDeviceToHost, s), "D2H");
  }
  CK(cudaEventRecord(ctx->ev[3], s), "event");
  CK(cudaStreamSynchronize(s), "solve");
  Ctl h;
  std::memcpy(&h, hp, sizeof(Ctl));
  const int32_t* ma = reinterpret_cast<const int32_t*>(hp + o_ma);
  const int32_t* mb = reinterpret_cast<const int32_t*>(hp + o_mb);
  const int32_t* yb = reinterpret_cast<const int32_t*>(hp + o_yb);
  const uint8_t* tbytes = reinterpret_cast<const uint8_t*>(hp + o_t);
  if (hout) *hout = h;
  const int64_t phases = h.phase;
  if (r->free_counts && r->free_cap > 0 && phases > 0) {
    const int64_t nf = std::min<int64_t>(phases, r->free_cap);
    const int64_t n1 = std::min<int64_t>(nf, fc_first);
    std::memcpy(r->free_counts, hp + o_fc, n1 * 8);
    if (nf > n1) {
      CK(cudaMemcpyAsync(r->free_counts + n1, ctx->fc.as<int64_t>() + n1, (nf - n1) * 8,
                         cudaMemcpyDeviceToHost, s), "D2H");
      CK(cudaStreamSynchronize(s), "D2H free_counts");
    }
  }
  // Back to the caller's orientation (assignment.cpp:395-399).
  if (!ctx->swapped) {
    std::memcpy(r->match_of_a, ma, ia * 4ull);
    std::memcpy(r->match_of_b, mb, ib * 4ull);
  } else {
    std::memcpy(r->match_of_a, mb, ib * 4ull);
    std::memcpy(r->match_of_b, ma, ia * 4ull);
  }
  if (r->y_a) {
    for (int i = 0; i < ia; ++i) {
      const int64_t t = ctx->width == 1   ? tbytes[i]
                        : ctx->width == 2 ? reinterpret_cast<const uint16_t*>(tbytes)[i]
                                          : reinterpret_cast<const uint32_t*>(tbytes)[i];
      r->y_a[i] = -t;
    }
  }
  if (r->y_b)
    for (int i = 0; i < ib; ++i) r->y_b[i] = yb[i];
  r->phases = phases;
  r->sum_ni = h.sum_ni;
  r->swapped = ctx->swapped;
  r->full_match_termination = h.full_match;
  double total = 0.0;  // matching_cost, core.cpp:95-102 (sequential over a: the reference's bits)
  const double* pc = reinterpret_cast<const double*>(hp + o_pc);
  for (int32_t a = 0; a < ctx->n_a; ++a) {
    const int32_t b = r->match_of_a[a];
    if (b != -1) total += dev_pc ? pc[a] : pair_cost(ctx, a, b);
  }
  r->cost = total;
  r->build_ms = ctx->build_ms;
  r->bytes_touched = static_cast<int64_t>(h.bytes_touched);
  r->bytes_alg = h.sum_ni * static_cast<int64_t>(ia) * ctx->width;
  r->width = ctx->width;
  for (int i = 0; i < 8; ++i) r->chain_stats[i] = static_cast<int64_t>(h.stat[i]);
  return OTPRG_OK;
}

int do_solve(otprg_ctx* ctx, otprg_result* r) {
  if (!r || !r->match_of_a || !r->match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  // init -> phase-1 propose scan (its own launch) -> phase loop (all phases)
  int st = do_begin(ctx, ctx->ev[0], ctx->ev[1], ctx->ev[7]);
  if (st) return st;
  cudaStream_t s = ctx->stream;
  if ((st = launch_loop(ctx, 0xffffffffu))) return st;
  CK(cudaEventRecord(ctx->ev[6], s), "event");
  if ((st = launch_finish(ctx))) return st;
  CK(cudaEventRecord(ctx->ev[2], s), "event");
  Ctl h{};
  if ((st = export_state(ctx, r, &h))) return st;
  if ((st = check_status(ctx, h, true))) return st;
  float ms_all = 0.f, ms_p1 = 0.f, ms_d2h = 0.f;
  cudaEventElapsedTime(&ms_all, ctx->ev[0], ctx->ev[2]);
  cudaEventElapsedTime(&ms_p1, ctx->ev[1], ctx->ev[7]);
  // the scan kernel's own device span (events around one launch also count
  // host enqueue gaps when the GPU runs ahead of the host)
  if (h.prop_t1 > h.prop_t0) ms_p1 = static_cast<float>((h.prop_t1 - h.prop_t0) * 1e-6);
  cudaEventElapsedTime(&ms_d2h, ctx->ev[0], ctx->ev[3]);
  float ms_loop = 0.f;
  cudaEventElapsedTime(&ms_loop, ctx->ev[7], ctx->ev[6]);
  r->loop_ms = ms_loop;
  r->solve_ms = ms_all;
  r->phase1_ms = ms_p1;
  r->solve_d2h_ms = ms_d2h;
  // init, phase-1 scan, loop (+ its tail launch), complete[, pair costs]
  r->gpu_launches = 3 + otprg::phase_loop_launches(ctx->width, ctx->smem_t, ctx->lda, ctx->loop_grid) +
                    (dev_pair_costs(ctx) ? 1 : 0);
  return OTPRG_OK;
}
}  // namespace otprg_capi

using namespace otprg_capi;

extern "C" {

int otprg_version(void) { return 1; }

int otprg_set_stream(otprg_ctx* ctx, void* stream) {
  if (!ctx) return OTPRG_PARAMETER;
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  CK(cudaStreamSynchronize(ctx->stream), "stream switch");
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  return OTPRG_OK;
}

int64_t otprg_scaled_floor(double c, double eps) { return host_scaled_floor(c, eps); }

int32_t otprg_points_threshold_table(double eps, double* thr, int32_t cap) {
  if (!(eps > 0.0 && eps < 1.0)) return -1;
  const int64_t uf = host_scaled_floor(1.0, eps);
  if (uf + 4 > std::numeric_limits<int32_t>::max()) return -1;
  const int32_t n = static_cast<int32_t>(uf + 2);
  if (!thr || cap < n) return n;
  const double sqrt2 = std::sqrt(2.0);
  // k(d2) = scaled_floor(sqrt(d2) / sqrt(2), eps) is monotone in d2, and d2 >= 0
  // is monotone in its bit pattern: bisect the bits for the first d2 at each level.
  auto k_of = [&](double d2) { return host_scaled_floor(std::sqrt(d2) / sqrt2, eps); };
  auto bits = [](double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; };
  auto from = [](uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; };
  const uint64_t top = bits(2.0);  // |a - b|^2 <= 2 for points of the unit square
  thr[0] = 0.0;
  for (int32_t j = 1; j < n; ++j) {
    if (k_of(from(top)) < j) {  // unreachable level
      thr[j] = std::numeric_limits<double>::infinity();
      continue;
    }
    uint64_t lo = 0, hi = top;  // k(from(hi)) >= j
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (k_of(from(mid)) >= j) hi = mid;
      else lo = mid + 1;
    }
    thr[j] = from(lo);
  }
  return n;
}

int otprg_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return OTPRG_DEVICE;
  size_t f = 0, t = 0;
  const cudaError_t e = cudaMemGetInfo(&f, &t);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return OTPRG_DEVICE;
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = t;
  return OTPRG_OK;
}

int otprg_create(int device, otprg_ctx** out) {
  if (!out) return OTPRG_PARAMETER;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return OTPRG_DEVICE;
  auto* ctx = new otprg_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return OTPRG_DEVICE;
  }
  ctx->own_stream = ctx->stream;
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  for (auto& e : ctx->timer) cudaEventCreate(&e);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  *out = ctx;
  return OTPRG_OK;
}

void otprg_destroy(otprg_ctx* ctx) {
  if (!ctx) return;
  for (otprg_ctx* c : ctx->multi) otprg_destroy(c);
  ctx->multi.clear();
  ctx->sh_plan.reset();  // graphs, exchange blocks and IPC mappings of a resident plan
  cudaSetDevice(ctx->device);
  for (DevBuf* b : {&ctx->kT, &ctx->t, &ctx->yb, &ctx->ma, &ctx->mb, &ctx->holder, &ctx->rowmin,
                    &ctx->lmeta, &ctx->lent, &ctx->lists, &ctx->mps, &ctx->fc, &ctx->ctl, &ctx->fa,
                    &ctx->fb, &ctx->stage, &ctx->pts, &ctx->flush, &ctx->trace, &ctx->sh_bounds,
                    &ctx->sh_pos, &ctx->sh_park[0], &ctx->sh_park[1], &ctx->sh_list, &ctx->v_out,
                    &ctx->v_k, &ctx->v_ya, &ctx->v_yb, &ctx->v_ma, &ctx->v_mb, &ctx->adm_cnt,
                    &ctx->adm_off, &ctx->adm_list, &ctx->ot_t, &ctx->ot_req, &ctx->ot_out,
                    &ctx->sk_K, &ctx->sk_P, &ctx->sk_vec, &ctx->sk_part, &ctx->sk_int})
    b->release();
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  for (auto& e : ctx->timer) cudaEventDestroy(e);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  if (ctx->ot_hpin) cudaFreeHost(ctx->ot_hpin);
  otprg::release_bounce(ctx);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* otprg_last_error(const otprg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int otprg_prepare(otprg_ctx* ctx, const otprg_problem* prob, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  int st = OTPRG_OK;
  if (!ctx->multi.empty()) {  // multi-device context: shard point instances
    if ((st = multi_prepare(ctx, prob))) return st;
    if (ctx->multi_prepared) {
      if (res) {
        res->build_ms = ctx->build_ms;
        res->width = ctx->multi[0]->width;
      }
      return OTPRG_OK;
    }
  }
  st = do_prepare(ctx, prob);
  if (st == OTPRG_OK && res) {
    res->build_ms = ctx->build_ms;
    res->width = ctx->width;
  }
  return st;
}

int otprg_solve_prepared(otprg_ctx* ctx, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (ctx->multi_prepared) return multi_solve(ctx, res);
  return do_solve(ctx, res);
}

int otprg_solve_assignment(otprg_ctx* ctx, const otprg_problem* prob, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->multi.empty()) {
    int st = multi_prepare(ctx, prob);
    if (st) return st;
    if (ctx->multi_prepared) return multi_solve(ctx, res);
  }
  int st = do_prepare(ctx, prob);
  if (st) return st;
  st = do_solve(ctx, res);
  if (st == OTPRG_OK) res->gpu_launches += ctx->build_launches;
  return st;
}

int otprg_scale_round_costs(otprg_ctx* ctx, const otprg_problem* prob, int32_t* k,
                            int32_t* unit_floor, int32_t* unit_ceil) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!k) return fail(ctx, OTPRG_PARAMETER, "k buffer is null");
  int st = do_prepare(ctx, prob);
  if (st) return st;
  const size_t total = static_cast<size_t>(ctx->n_a) * ctx->n_b;
  ctx->stage_holds_cost = false;
  CK(ctx->stage.ensure(std::max(ctx->stage.n, total * 4)), "alloc export");
  // the staging buffer may hold the dense input; it is no longer needed
  CK(otprg::launch_export_k(ctx->kT.p, ctx->ia, ctx->ib, ctx->lda, ctx->width, ctx->swapped,
                            ctx->stage.as<int32_t>(), ctx->stream),
     "export launch");
  CK(cudaMemcpyAsync(k, ctx->stage.p, total * 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H k");
  CK(cudaStreamSynchronize(ctx->stream), "export");
  if (unit_floor) *unit_floor = ctx->unit_floor;
  if (unit_ceil) *unit_ceil = ctx->unit_ceil;
  return OTPRG_OK;
}

int otprg_load_mnist_pair(const char* path, int32_t n, uint64_t seed, uint8_t* img_a,
                          uint8_t* img_b, char* err, int32_t err_cap) {
  auto fail_msg = [&](int code, const std::string& m) {
    if (err && err_cap > 0) {
      std::strncpy(err, m.c_str(), static_cast<size_t>(err_cap) - 1);
      err[err_cap - 1] = 0;
    }
    return code;
  };
  if (n < 1) return fail_msg(OTPRG_PARAMETER, "load_mnist_pair: n must be >= 1");
  if (!path || !img_a || !img_b) return fail_msg(OTPRG_PARAMETER, "null argument");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail_msg(OTPRG_INPUT, std::string("cannot open image file: ") + path);
  std::vector<unsigned char> bytes;
  {
    unsigned char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) bytes.insert(bytes.end(), buf, buf + got);
    std::fclose(f);
  }
  auto be32 = [](const unsigned char* p) {
    return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
  };
  // instances.cpp:88-103
  if (bytes.size() < 16) return fail_msg(OTPRG_INPUT, "image file too short for a header");
  if (be32(bytes.data()) != 0x00000803) return fail_msg(OTPRG_INPUT, "bad IDX3 magic: expected 0x00000803");
  const uint32_t count = be32(bytes.data() + 4);
  if (be32(bytes.data() + 8) != 28 || be32(bytes.data() + 12) != 28)
    return fail_msg(OTPRG_INPUT, "unexpected image dimensions: want 28x28");
  const size_t pixels = 28 * 28;
  if (bytes.size() < 16 + static_cast<size_t>(count) * pixels)
    return fail_msg(OTPRG_INPUT, "image file truncated");
  if (count < static_cast<uint32_t>(2 * n))
    return fail_msg(OTPRG_INPUT, "not enough images: need " + std::to_string(2 * n) +
                                     ", file has " + std::to_string(count));
  // seeded sample of 2n distinct indices, partial Fisher-Yates (instances.cpp:105-112)
  auto splitmix64 = [](uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  std::mt19937_64 rng(splitmix64(seed ^ 0xD1B54A32D192ED03ULL));
  auto bounded = [&](uint64_t m) {  // instances.cpp:25-32
    const uint64_t limit = ~uint64_t{0} - (~uint64_t{0}) % m;
    uint64_t x;
    do {
      x = rng();
    } while (x >= limit);
    return x % m;
  };
  std::vector<uint32_t> pool(count);
  for (uint32_t i = 0; i < count; ++i) pool[i] = i;
  for (int32_t i = 0; i < 2 * n; ++i) {
    const uint64_t j = static_cast<uint64_t>(i) + bounded(count - static_cast<uint64_t>(i));
    std::swap(pool[i], pool[j]);
  }
  for (int32_t i = 0; i < 2 * n; ++i) {
    const unsigned char* src = bytes.data() + 16 + static_cast<size_t>(pool[i]) * pixels;
    size_t total = 0;
    for (size_t p = 0; p < pixels; ++p) total += src[p];
    if (total == 0)  // instances.cpp:121-123
      return fail_msg(OTPRG_INPUT, "image " + std::to_string(pool[i]) + " has zero total intensity");
    std::memcpy((i < n ? img_a + static_cast<size_t>(i) * pixels
                       : img_b + static_cast<size_t>(i - n) * pixels),
                src, pixels);
  }
  return OTPRG_OK;
}

int otprg_uniform_square_points(int32_t n, uint64_t seed, double* pts_a, double* pts_b) {
  if (n < 1 || !pts_a || !pts_b) return OTPRG_PARAMETER;
  auto splitmix64 = [](uint64_t x) {  // instances.cpp:41-46
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  auto u01 = [](std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; };
  std::mt19937_64 ra(splitmix64(seed));
  std::mt19937_64 rb(splitmix64(seed ^ 0x9E3779B97F4A7C15ULL));
  for (int32_t i = 0; i < n; ++i) {
    pts_a[2 * static_cast<size_t>(i)] = u01(ra);
    pts_a[2 * static_cast<size_t>(i) + 1] = u01(ra);
  }
  for (int32_t i = 0; i < n; ++i) {
    pts_b[2 * static_cast<size_t>(i)] = u01(rb);
    pts_b[2 * static_cast<size_t>(i) + 1] = u01(rb);
  }
  return OTPRG_OK;
}

int otprg_begin(otprg_ctx* ctx) {
  if (!ctx) return OTPRG_PARAMETER;
  return do_begin(ctx);
}

int otprg_step(otprg_ctx* ctx, int64_t max_phases, int64_t* phases_done, int32_t* finished) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun || ctx->completed) return fail(ctx, OTPRG_PARAMETER, "otprg_begin() first");
  const uint32_t cap = max_phases <= 0 || max_phases > 0xfffffffe ? 0xffffffffu
                                                                  : static_cast<uint32_t>(max_phases);
  int st = launch_loop(ctx, cap);
  if (st) return st;
  Ctl h{};
  CK(cudaMemcpyAsync(&h, ctx->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream), "D2H ctl");
  CK(cudaStreamSynchronize(ctx->stream), "step");
  if ((st = check_status(ctx, h, false))) return st;
  if (phases_done) *phases_done = h.phase;
  if (finished) *finished = h.done;
  return OTPRG_OK;
}

int otprg_snapshot(otprg_ctx* ctx, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun) return fail(ctx, OTPRG_PARAMETER, "otprg_begin() first");
  if (!res || !res->match_of_a || !res->match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  Ctl h{};
  int st = export_state(ctx, res, &h);
  if (st) return st;
  return check_status(ctx, h, false);
}

int otprg_finish(otprg_ctx* ctx, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->begun) return fail(ctx, OTPRG_PARAMETER, "otprg_begin() first");
  if (!res || !res->match_of_a || !res->match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  int st = launch_loop(ctx, 0xffffffffu);  // run any remaining phases
  if (st) return st;
  if (!ctx->completed && (st = launch_finish(ctx))) return st;
  Ctl h{};
  if ((st = export_state(ctx, res, &h))) return st;
  return check_status(ctx, h, true);
}

int otprg_set_trace(otprg_ctx* ctx, int64_t max_phases) {
  if (!ctx) return OTPRG_PARAMETER;
  if (max_phases <= 0) {
    ctx->trace_cap = 0;
    return OTPRG_OK;
  }
  const uint32_t cap = static_cast<uint32_t>(std::min<int64_t>(max_phases, 1 << 22));
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  CK(ctx->trace.ensure(cap * 8ull * otprg::kTraceSlots), "alloc trace");
  ctx->trace_cap = cap;
  return OTPRG_OK;
}

int otprg_get_trace(otprg_ctx* ctx, uint64_t* out, int64_t max_phases) {
  if (!ctx || !out) return OTPRG_PARAMETER;
  if (!ctx->trace_cap) return fail(ctx, OTPRG_PARAMETER, "tracing is off");
  const int64_t n = std::min<int64_t>(max_phases, ctx->trace_cap);
  CK(cudaMemcpyAsync(out, ctx->trace.p, n * 8 * otprg::kTraceSlots, cudaMemcpyDeviceToHost, ctx->stream), "D2H trace");
  CK(cudaStreamSynchronize(ctx->stream), "trace");
  return OTPRG_OK;
}

int otprg_timer_start(otprg_ctx* ctx) {
  if (!ctx) return OTPRG_PARAMETER;
  CK(cudaEventRecord(ctx->timer[0], ctx->stream), "timer");
  return OTPRG_OK;
}

int otprg_timer_stop(otprg_ctx* ctx, double* ms) {
  if (!ctx || !ms) return OTPRG_PARAMETER;
  CK(cudaEventRecord(ctx->timer[1], ctx->stream), "timer");
  CK(cudaEventSynchronize(ctx->timer[1]), "timer");
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]), "timer");
  *ms = f;
  return OTPRG_OK;
}

int otprg_flush_l2(otprg_ctx* ctx) {
  if (!ctx) return OTPRG_PARAMETER;
  const size_t bytes = 256ull << 20;
  CK(ctx->flush.ensure(bytes), "alloc flush");
  CK(otprg::launch_flush(ctx->flush.p, bytes, ctx->stream), "flush launch");
  CK(cudaStreamSynchronize(ctx->stream), "flush");
  return OTPRG_OK;
}

}  // extern "C"

// ---- invariant suite --------------------------------
namespace {

struct VerifyResult {
  unsigned long long first, count;
};

int run_verify(otprg_ctx* ctx, bool host_state, int n_a, int n_b, long long bound,
               VerifyResult* r) {
  CK(ctx->v_out.ensure(sizeof(otprg::VerifyOut)), "alloc verify");
  otprg::VerifyOut init{~0ull, 0ull};
  auto* out = ctx->v_out.as<otprg::VerifyOut>();
  CK(cudaMemcpyAsync(out, &init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream), "H2D verify");
  if (host_state)
    CK(otprg::launch_verify_host(ctx->v_k.as<int32_t>(), ctx->v_ya.as<long long>(),
                                 ctx->v_yb.as<long long>(), ctx->v_ma.as<int32_t>(),
                                 ctx->v_mb.as<int32_t>(), n_a, n_b, bound, out, ctx->stream),
       "verify launch");
  else
    CK(otprg::launch_verify_state(ctx->kT.p, ctx->lda, ctx->width, ctx->t.p, ctx->yb.as<int32_t>(),
                                  ctx->ma.as<int32_t>(), ctx->mb.as<int32_t>(), n_a, n_b, bound, out,
                                  ctx->stream),
       "verify launch");
  otprg::VerifyOut h{};
  CK(cudaMemcpyAsync(&h, out, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream), "D2H verify");
  CK(cudaStreamSynchronize(ctx->stream), "verify");
  r->first = h.first;
  r->count = h.count;
  return OTPRG_OK;
}

// Splits the first-violation key; dual/edge values come from `get`.
template <typename Get>
void decode_violation(const VerifyResult& r, int n_a, int n_b, Get get, otprg_feasibility* f) {
  f->violations = 0;
  f->kind = OTPRG_VIOL_NONE;
  f->a = f->b = -1;
  f->pad = 0;
  f->sum = f->k = 0;
  if (r.first == ~0ull) return;
  const unsigned section = static_cast<unsigned>(r.first >> 60);
  const unsigned long long index = (r.first >> 4) & ((1ull << 56) - 1);
  f->kind = static_cast<int32_t>(r.first & 15);
  f->violations = section == 0 ? 1 : static_cast<int64_t>(r.count);  // validate() stops the check
  if (section == 0) {
    if (f->kind == OTPRG_VIOL_MATCH_A) f->a = static_cast<int32_t>(index);
    else f->b = static_cast<int32_t>(index - n_a);
  } else if (section == 1) {
    f->a = static_cast<int32_t>(index);
  } else if (section == 2) {
    f->b = static_cast<int32_t>(index);
  } else {
    f->a = static_cast<int32_t>(index / n_b);
    f->b = static_cast<int32_t>(index % n_b);
  }
  get(f);
}

}  // namespace

extern "C" {

int otprg_verify_feasibility(otprg_ctx* ctx, otprg_feasibility* out) {
  if (!ctx || !out) return OTPRG_PARAMETER;
  if (!ctx->begun || ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_begin() first");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  VerifyResult r{};
  int st = run_verify(ctx, false, ctx->ia, ctx->ib, static_cast<long long>(ctx->unit_ceil) + 2, &r);
  if (st) return st;
  int err = 0;
  decode_violation(r, ctx->ia, ctx->ib,
                   [&](otprg_feasibility* f) {
                     uint32_t tv = 0;  // w low bytes (little endian), rest zero
                     int32_t ybv = 0;
                     uint32_t kv = 0;
                     const int w = ctx->width;
                     if (f->a >= 0 && cudaMemcpy(&tv, static_cast<char*>(ctx->t.p) + static_cast<size_t>(f->a) * w, w,
                                                 cudaMemcpyDeviceToHost) != cudaSuccess) err = 1;
                     if (f->b >= 0 && cudaMemcpy(&ybv, ctx->yb.as<int32_t>() + f->b, 4,
                                                 cudaMemcpyDeviceToHost) != cudaSuccess) err = 1;
                     if (f->a >= 0 && f->b >= 0 &&
                         cudaMemcpy(&kv, static_cast<char*>(ctx->kT.p) +
                                             (static_cast<size_t>(f->b) * ctx->lda + f->a) * w,
                                    w, cudaMemcpyDeviceToHost) != cudaSuccess) err = 1;
                     const long long ya = -static_cast<long long>(tv);
                     const long long kk = kv;
                     if (f->kind >= OTPRG_VIOL_NOT_TIGHT) {
                       f->sum = ya + ybv;
                       f->k = kk;
                     } else if (f->kind >= OTPRG_VIOL_SUPPLY_NEGATIVE) {
                       f->sum = ybv;
                     } else if (f->kind >= OTPRG_VIOL_DEMAND_POSITIVE) {
                       f->sum = ya;
                     }
                   },
                   out);
  if (err) return fail(ctx, OTPRG_DEVICE, "D2H of the violation details failed");
  return OTPRG_OK;
}

int otprg_verify_result(otprg_ctx* ctx, const int64_t* y_a, const int64_t* y_b, const int32_t* match_of_a,
                        const int32_t* match_of_b, otprg_feasibility* out) {
  if (!ctx || !out) return OTPRG_PARAMETER;
  if (!ctx->prepared || ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_prepare() first");
  if (!y_a || !y_b || !match_of_a || !match_of_b) return fail(ctx, OTPRG_PARAMETER, "null state");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int ia = ctx->ia, ib = ctx->ib, w = ctx->width;
  // the solver's own representation: t(a) = -Y(a) in the storage type, Y(b) int32
  const int64_t tmax = otprg::storage_tmax(w);
  std::vector<uint8_t> t(static_cast<size_t>(ctx->lda) * w, 0);
  std::vector<int32_t> yb(ib);
  for (int a = 0; a < ia; ++a) {
    if (y_a[a] > 0 || -y_a[a] > tmax)
      return fail(ctx, OTPRG_PARAMETER, "demand dual outside the device representation at a=" + std::to_string(a));
    const uint32_t v = static_cast<uint32_t>(-y_a[a]);
    std::memcpy(t.data() + static_cast<size_t>(a) * w, &v, w);  // little endian: low w bytes
  }
  for (int b = 0; b < ib; ++b) {
    if (y_b[b] < 0 || y_b[b] > tmax)
      return fail(ctx, OTPRG_PARAMETER, "supply dual outside the device representation at b=" + std::to_string(b));
    yb[b] = static_cast<int32_t>(y_b[b]);
  }
  CK(ctx->v_ya.ensure(t.size()), "alloc");
  CK(ctx->v_yb.ensure(ib * 4ull), "alloc");
  CK(ctx->v_ma.ensure(ia * 4ull), "alloc");
  CK(ctx->v_mb.ensure(ib * 4ull), "alloc");
  CK(cudaMemcpyAsync(ctx->v_ya.p, t.data(), t.size(), cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_yb.p, yb.data(), ib * 4ull, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_ma.p, match_of_a, ia * 4ull, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_mb.p, match_of_b, ib * 4ull, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(ctx->v_out.ensure(sizeof(otprg::VerifyOut)), "alloc verify");
  otprg::VerifyOut init{~0ull, 0ull};
  auto* vo = ctx->v_out.as<otprg::VerifyOut>();
  CK(cudaMemcpyAsync(vo, &init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream), "H2D verify");
  CK(otprg::launch_verify_state(ctx->kT.p, ctx->lda, w, ctx->v_ya.p, ctx->v_yb.as<int32_t>(),
                                ctx->v_ma.as<int32_t>(), ctx->v_mb.as<int32_t>(), ia, ib,
                                static_cast<long long>(ctx->unit_ceil) + 2, vo, ctx->stream),
     "verify launch");
  otprg::VerifyOut h{};
  CK(cudaMemcpyAsync(&h, vo, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream), "D2H verify");
  CK(cudaStreamSynchronize(ctx->stream), "verify");
  VerifyResult r{h.first, h.count};
  int err = 0;
  decode_violation(r, ia, ib,
                   [&](otprg_feasibility* f) {
                     uint32_t kv = 0;
                     if (f->a >= 0 && f->b >= 0 &&
                         cudaMemcpy(&kv, static_cast<char*>(ctx->kT.p) +
                                             (static_cast<size_t>(f->b) * ctx->lda + f->a) * w,
                                    w, cudaMemcpyDeviceToHost) != cudaSuccess) err = 1;
                     if (f->kind >= OTPRG_VIOL_NOT_TIGHT) {
                       f->sum = y_a[f->a] + y_b[f->b];
                       f->k = kv;
                     } else if (f->kind >= OTPRG_VIOL_SUPPLY_NEGATIVE) {
                       f->sum = y_b[f->b];
                     } else if (f->kind >= OTPRG_VIOL_DEMAND_POSITIVE) {
                       f->sum = y_a[f->a];
                     }
                   },
                   out);
  if (err) return fail(ctx, OTPRG_DEVICE, "D2H of the violation details failed");
  return OTPRG_OK;
}

int otprg_verify_host(otprg_ctx* ctx, int32_t n_a, int32_t n_b, const int32_t* k, int32_t unit_ceil,
                      const int64_t* y_a, const int64_t* y_b, const int32_t* match_of_a,
                      const int32_t* match_of_b, otprg_feasibility* out) {
  if (!ctx || !out) return OTPRG_PARAMETER;
  if (n_a < 1 || n_b < 1 || !k || !y_a || !y_b || !match_of_a || !match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "null or empty state");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  const size_t na = n_a, nb = n_b;
  CK(ctx->v_k.ensure(na * nb * 4), "alloc");
  CK(ctx->v_ya.ensure(na * 8), "alloc");
  CK(ctx->v_yb.ensure(nb * 8), "alloc");
  CK(ctx->v_ma.ensure(na * 4), "alloc");
  CK(ctx->v_mb.ensure(nb * 4), "alloc");
  CK(cudaMemcpyAsync(ctx->v_k.p, k, na * nb * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_ya.p, y_a, na * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_yb.p, y_b, nb * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_ma.p, match_of_a, na * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->v_mb.p, match_of_b, nb * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  VerifyResult r{};
  int st = run_verify(ctx, true, n_a, n_b, static_cast<long long>(unit_ceil) + 2, &r);
  if (st) return st;
  decode_violation(r, n_a, n_b,
                   [&](otprg_feasibility* f) {
                     if (f->kind >= OTPRG_VIOL_NOT_TIGHT) {
                       f->sum = y_a[f->a] + y_b[f->b];
                       f->k = k[static_cast<size_t>(f->a) * nb + f->b];
                     } else if (f->kind >= OTPRG_VIOL_SUPPLY_NEGATIVE) {
                       f->sum = y_b[f->b];
                     } else if (f->kind >= OTPRG_VIOL_DEMAND_POSITIVE) {
                       f->sum = y_a[f->a];
                     }
                   },
                   out);
  return OTPRG_OK;
}

int otprg_admissible(otprg_ctx* ctx, int32_t* b_free, int64_t* offsets, int32_t* a_list,
                     int64_t a_cap, int64_t* n_free, int64_t* n_edges) {
  if (!ctx || !b_free || !offsets) return OTPRG_PARAMETER;
  if (!ctx->begun || ctx->sharded) return fail(ctx, OTPRG_PARAMETER, "otprg_begin() first");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int ib = ctx->ib;
  CK(ctx->adm_cnt.ensure((static_cast<size_t>(ib) + 1) * 8), "alloc");
  CK(ctx->adm_off.ensure((static_cast<size_t>(ib) + 1) * 8), "alloc");
  int* d_count = reinterpret_cast<int*>(ctx->adm_cnt.as<long long>() + ib);
  CK(otprg::launch_free_list(ctx->mb.as<int32_t>(), ib, ctx->fb.as<int32_t>(), d_count, ctx->stream),
     "free list launch");
  int nf = 0;
  CK(cudaMemcpyAsync(&nf, d_count, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  CK(cudaStreamSynchronize(ctx->stream), "free list");
  CK(otprg::launch_admissible(ctx->kT.p, ctx->lda, ctx->width, ctx->t.p, ctx->yb.as<int32_t>(),
                              ctx->fb.as<int32_t>(), nf, ctx->ia, ctx->adm_cnt.as<long long>(), nullptr,
                              nullptr, ctx->stream),
     "admissible count launch");
  std::vector<long long> cnt(static_cast<size_t>(nf));
  if (nf > 0) {
    CK(cudaMemcpyAsync(cnt.data(), ctx->adm_cnt.p, static_cast<size_t>(nf) * 8, cudaMemcpyDeviceToHost,
                       ctx->stream), "D2H");
    CK(cudaMemcpyAsync(b_free, ctx->fb.p, static_cast<size_t>(nf) * 4, cudaMemcpyDeviceToHost,
                       ctx->stream), "D2H");
  }
  CK(cudaStreamSynchronize(ctx->stream), "admissible count");
  offsets[0] = 0;
  for (int i = 0; i < nf; ++i) offsets[i + 1] = offsets[i] + cnt[i];
  const int64_t total = offsets[nf];
  if (n_free) *n_free = nf;
  if (n_edges) *n_edges = total;
  if (!a_list || a_cap < total || total == 0) return OTPRG_OK;
  CK(ctx->adm_list.ensure(static_cast<size_t>(total) * 4), "alloc");
  static_assert(sizeof(long long) == sizeof(int64_t), "offsets");
  CK(cudaMemcpyAsync(ctx->adm_off.p, offsets, (static_cast<size_t>(nf) + 1) * 8, cudaMemcpyHostToDevice,
                     ctx->stream), "H2D");
  CK(otprg::launch_admissible(ctx->kT.p, ctx->lda, ctx->width, ctx->t.p, ctx->yb.as<int32_t>(),
                              ctx->fb.as<int32_t>(), nf, ctx->ia, nullptr, ctx->adm_off.as<long long>(),
                              ctx->adm_list.as<int32_t>(), ctx->stream),
     "admissible fill launch");
  CK(cudaMemcpyAsync(a_list, ctx->adm_list.p, static_cast<size_t>(total) * 4, cudaMemcpyDeviceToHost,
                     ctx->stream), "D2H");
  CK(cudaStreamSynchronize(ctx->stream), "admissible");
  return OTPRG_OK;
}

}  // extern "C"

// ---- copy mode --------------------------------------
namespace {

// Mirror of the host-side loop state into the device control block, so
// otprg_snapshot / otprg_verify_feasibility / export_state see copy-mode runs
// exactly like fused ones.
int groups_publish(otprg_ctx* ctx) {
  Ctl* d = ctx->ctl.as<Ctl>();
  const uint32_t ph = ctx->g_phase;
  const int32_t done = ctx->g_done ? 1 : 0, full = ctx->g_full ? 1 : 0;
  CK(cudaMemcpyAsync(&d->phase, &ph, 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(&d->sum_ni, &ctx->g_sum_ni, 8, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(&d->done, &done, 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(&d->full_match, &full, 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  if (ph > 0 && static_cast<int64_t>(ph) <= ctx->fc_cap)
    CK(cudaMemcpyAsync(ctx->fc.as<int64_t>() + ph - 1, &ctx->g_fc[ph - 1], 8, cudaMemcpyHostToDevice,
                       ctx->stream), "H2D");
  CK(cudaStreamSynchronize(ctx->stream), "publish");  // (host sources live on the stack)
  return OTPRG_OK;
}

}  // namespace

extern "C" {

int otprg_groups_begin(otprg_ctx* ctx, const otprg_problem* p, const int32_t* demand_groups,
                       const int32_t* supply_groups) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!p || !demand_groups || !supply_groups)
    return fail(ctx, OTPRG_PARAMETER, "copy mode needs both demand and supply groups");
  if (p->n_b > p->n_a) return fail(ctx, OTPRG_PARAMETER, "copy mode requires n_b <= n_a");
  if (p->n_a >= (1 << 21)) return fail(ctx, OTPRG_PARAMETER, "copy mode supports n_a < 2^21");
  int dmax = -1, smax = -1;
  for (int32_t a = 0; a < p->n_a; ++a) {
    if (demand_groups[a] < 0 || demand_groups[a] >= (1 << 21))
      return fail(ctx, OTPRG_PARAMETER, "group ids must lie in [0, 2^21)");
    dmax = std::max(dmax, demand_groups[a]);
  }
  for (int32_t b = 0; b < p->n_b; ++b) {
    if (supply_groups[b] < 0 || supply_groups[b] >= (1 << 21))
      return fail(ctx, OTPRG_PARAMETER, "group ids must lie in [0, 2^21)");
    smax = std::max(smax, supply_groups[b]);
  }
  int st = do_prepare(ctx, p);
  if (st) return st;
  if ((st = do_begin(ctx))) return st;
  const size_t na = ctx->ia, nb = ctx->ib;
  ctx->g_ndg = dmax + 1;
  ctx->g_nsg = smax + 1;
  CK(ctx->g_d.ensure(na * 4), "alloc");
  CK(ctx->g_s.ensure(nb * 4), "alloc");
  CK(ctx->g_keys.ensure(na * 8), "alloc");
  CK(ctx->g_keys2.ensure(na * 8), "alloc");
  CK(ctx->g_vals.ensure(na * 4), "alloc");
  CK(ctx->g_pi.ensure(na * 4), "alloc");
  CK(ctx->g_rank.ensure(na * 4), "alloc");
  CK(ctx->g_tmp.ensure(std::max<size_t>(otprg::copy_sort_temp_bytes(ctx->ia), 16)), "alloc");
  CK(ctx->g_gmax.ensure(static_cast<size_t>(ctx->g_nsg) * 4), "alloc");
  CK(ctx->g_cnt.ensure(16), "alloc");
  CK(cudaMemcpyAsync(ctx->g_d.p, demand_groups, na * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  CK(cudaMemcpyAsync(ctx->g_s.p, supply_groups, nb * 4, cudaMemcpyHostToDevice, ctx->stream), "H2D");
  ctx->groups_mode = true;
  ctx->g_done = ctx->g_full = false;
  ctx->g_phase = 0;
  ctx->g_sum_ni = 0;
  ctx->g_fc.clear();
  return groups_publish(ctx);
}

// One phase of solve_oriented (assignment.cpp:316-364) in copy mode.
int otprg_groups_step(otprg_ctx* ctx, int64_t* phases_done, int32_t* finished) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!ctx->groups_mode || !ctx->begun) return fail(ctx, OTPRG_PARAMETER, "otprg_groups_begin() first");
  cudaStream_t s = ctx->stream;
  if (!ctx->g_done) {
    int* d_count = ctx->g_cnt.as<int>() + 1;
    CK(otprg::launch_free_list(ctx->mb.as<int32_t>(), ctx->ib, ctx->fb.as<int32_t>(), d_count, s),
       "free list");
    int nf = 0;
    CK(cudaMemcpyAsync(&nf, d_count, 4, cudaMemcpyDeviceToHost, s), "D2H");
    CK(cudaStreamSynchronize(s), "free list");
    const double threshold = ctx->eps * static_cast<double>(std::min(ctx->n_a, ctx->n_b));
    if (static_cast<double>(nf) <= threshold) {
      ctx->g_done = true;
      ctx->g_full = nf == 0;
    } else {
      const int64_t cap = static_cast<int64_t>(std::ceil((1.0 + 2.0 * ctx->eps) / (ctx->eps * ctx->eps))) + 8;
      ctx->g_phase += 1;
      ctx->g_fc.push_back(nf);
      ctx->g_sum_ni += nf;
      CK(otprg::copy_order(ctx->g_d.as<int32_t>(), ctx->g_s.as<int32_t>(), ctx->ma.as<int32_t>(), ctx->ia,
                           ctx->g_keys.as<unsigned long long>(), ctx->g_keys2.as<unsigned long long>(),
                           ctx->g_vals.as<int32_t>(), ctx->g_pi.as<int32_t>(), ctx->g_rank.as<int32_t>(),
                           ctx->g_tmp.p, ctx->g_tmp.n, s),
         "copy order");
      int* mp_cnt = ctx->g_cnt.as<int>();
      CK(cudaMemsetAsync(mp_cnt, 0, 4, s), "memset");
      unsigned long long* holder = ctx->holder.as<unsigned long long>();
      CK(otprg::copy_da(ctx->kT.p, ctx->lda, ctx->width, ctx->t.p, ctx->yb.as<int32_t>(), ctx->ma.as<int32_t>(),
                        holder, ctx->g_pi.as<int32_t>(), ctx->g_rank.as<int32_t>(), ctx->fb.as<int32_t>(), nf,
                        ctx->ia, ctx->g_phase, ctx->mps.as<int2>(), mp_cnt, ctx->ctl.as<Ctl>(), s),
         "copy DA");
      CK(otprg::copy_apply(ctx->mps.as<int2>(), mp_cnt, holder, ctx->ma.as<int32_t>(), ctx->mb.as<int32_t>(),
                           ctx->t.p, ctx->width, ctx->g_phase, ctx->ctl.as<Ctl>(), s),
         "copy apply");
      CK(otprg::copy_lift(ctx->yb.as<int32_t>(), ctx->mb.as<int32_t>(), ctx->g_s.as<int32_t>(), ctx->ib,
                          ctx->g_nsg, ctx->g_gmax.as<int>(), s),
         "copy lift");
      Ctl h{};
      CK(cudaMemcpyAsync(&h, ctx->ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost, s), "D2H ctl");
      CK(cudaStreamSynchronize(s), "copy phase");
      int st = check_status(ctx, h, false);
      if (st) return st;
      if (static_cast<int64_t>(ctx->g_phase) > cap)
        return fail(ctx, OTPRG_INVARIANT, "phase count exceeded the proven bound; solver state is corrupt");
    }
    int st = groups_publish(ctx);
    if (st) return st;
  }
  if (phases_done) *phases_done = ctx->g_phase;
  if (finished) *finished = ctx->g_done ? 1 : 0;
  return OTPRG_OK;
}

int otprg_groups_finish(otprg_ctx* ctx, otprg_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!res || !res->match_of_a || !res->match_of_b)
    return fail(ctx, OTPRG_PARAMETER, "result buffers are null");
  int32_t fin = 0;
  while (!fin) {
    int st = otprg_groups_step(ctx, nullptr, &fin);
    if (st) return st;
  }
  int st = launch_finish(ctx);
  if (st) return st;
  Ctl h{};
  if ((st = export_state(ctx, res, &h))) return st;
  res->gpu_launches = 0;
  ctx->groups_mode = false;
  return check_status(ctx, h, true);
}

}  // extern "C"

