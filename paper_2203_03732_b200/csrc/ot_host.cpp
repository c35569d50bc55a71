// ot_host.cpp — optimal transport through the copy/cluster phase algorithm
// (reference: solve_ot, src/ot.cpp:705-732; scale_and_round :109-128;
// solve_copy_matching :418-637; plan_from_flow :639-703).
//
// Division of labour:
//   device  rounding of the dense cost at eps/3 into kT (K1, cost_kernels.cu)
//           and the whole phase (ot_device.cu): free list, admissible
//           clusters of every free supply vertex, the claim step as a
//           capacitated deferred acceptance (K10), the cluster updates and
//           normalisation (K11) — the cluster state never leaves the device;
//   host    the phase loop's control (a few synchronisations per phase: the
//           termination test, buffer sizes, the DA rounds), the completion
//           and plan_from_flow on the final sparse flow, and the debug hooks
//           (check_invariants / observer) on an exported copy of the state.
// All floating-point operations of plan_from_flow run in the reference's
// order on the nonzero entries only, so the plan's masses and cost are
// bit-equal.
#include <algorithm>
#include <array>
#include <chrono>
#include <random>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <utility>
#include <vector>

#include "ctx.h"
#include "kernels.h"

namespace {

using otprg::DevBuf;
using otprg::host_scaled_floor;

constexpr double kMassTolerance = 1e-9;  // ot.cpp:15

struct OtError {
  int code;
  std::string msg;
};

int64_t exact_floor(double x) {  // ot.cpp:17-22
  auto f = static_cast<int64_t>(std::floor(x));
  while (static_cast<double>(f + 1) <= x) ++f;
  while (static_cast<double>(f) > x) --f;
  return f;
}

int64_t exact_ceil(double x) {  // ot.cpp:24-29
  auto c = static_cast<int64_t>(std::ceil(x));
  while (static_cast<double>(c - 1) >= x) --c;
  while (static_cast<double>(c) < x) ++c;
  return c;
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
};

#define OT_CK(expr, what)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw OtError{OTPRG_DEVICE, std::string(what) + ": " + cudaGetErrorString(_e)}; \
  } while (0)

void validate_ot(const otprg_ot_problem* p) {  // OTInstance::validate, ot.cpp:62-89 (masses)
  if (!p || p->n_a < 1 || p->n_b < 1)
    throw OtError{OTPRG_PARAMETER, "OT instance needs at least one point per side"};
  if (!p->mu || !p->nu || !p->cost) throw OtError{OTPRG_PARAMETER, "null instance pointer"};
  double sum_mu = 0.0, sum_nu = 0.0;
  for (int32_t a = 0; a < p->n_a; ++a) {
    if (!(p->mu[a] >= 0.0)) throw OtError{OTPRG_PARAMETER, "negative or NaN demand mass"};
    sum_mu += p->mu[a];
  }
  for (int32_t b = 0; b < p->n_b; ++b) {
    if (!(p->nu[b] >= 0.0)) throw OtError{OTPRG_PARAMETER, "negative or NaN supply mass"};
    sum_nu += p->nu[b];
  }
  if (std::abs(sum_mu - 1.0) > kMassTolerance || std::abs(sum_nu - 1.0) > kMassTolerance)
    throw OtError{OTPRG_INPUT, "masses must each sum to 1 within 1e-9 (got " + std::to_string(sum_mu) +
                                   " and " + std::to_string(sum_nu) + ")"};
}

struct ScaledMasses {
  double theta = 0.0;
  std::vector<int64_t> d, s;
  int64_t total_d = 0, total_s = 0;
};

ScaledMasses scale_and_round(const otprg_ot_problem* p, double eps) {  // ot.cpp:109-128
  if (!(eps > 0.0 && eps < 1.0)) throw OtError{OTPRG_PARAMETER, "eps must lie in (0, 1)"};
  const auto n = static_cast<double>(std::max(p->n_a, p->n_b));
  ScaledMasses sm;
  sm.theta = 4.0 * n / eps;
  if (!(sm.theta < 4.0e15))
    throw OtError{OTPRG_PARAMETER, "theta = 4n/eps too large: copy counts overflow"};
  sm.d.resize(p->n_a);
  sm.s.resize(p->n_b);
  for (int32_t a = 0; a < p->n_a; ++a) sm.total_d += (sm.d[a] = exact_ceil(p->mu[a] * sm.theta));
  for (int32_t b = 0; b < p->n_b; ++b) sm.total_s += (sm.s[b] = exact_floor(p->nu[b] * sm.theta));
  if (sm.total_s > sm.total_d)
    throw OtError{OTPRG_INVARIANT, "scaled supplies exceed scaled demands"};
  return sm;
}

// ---- flat ClusterState (otprg_cluster_state) and the reference's checks ----

struct FlatState {
  int32_t n_a = 0, n_b = 0;
  std::vector<int32_t> dem_off, flow_b, sup_off;
  std::vector<int64_t> dem_y, dem_free, flow_off, flow_cnt, sup_y, sup_free, sup_matched;

  otprg_cluster_state view() const {
    return otprg_cluster_state{n_a,          n_b,          dem_off.data(), dem_y.data(),  dem_free.data(),
                               flow_off.data(), flow_b.data(), flow_cnt.data(), sup_off.data(), sup_y.data(),
                               sup_free.data(), sup_matched.data()};
  }
  // ClusterState::sum_abs_duals (ot.cpp:181-188)
  int64_t sum_abs_duals() const {
    int64_t t = 0;
    for (size_t c = 0; c < dem_y.size(); ++c) {
      int64_t cnt = dem_free[c];
      for (int64_t f = flow_off[c]; f < flow_off[c + 1]; ++f) cnt += flow_cnt[f];
      t += std::llabs(dem_y[c]) * cnt;
    }
    for (size_t c = 0; c < sup_y.size(); ++c) t += std::llabs(sup_y[c]) * (sup_free[c] + sup_matched[c]);
    return t;
  }
};

// check_cluster_invariant (ot.cpp:190-265) on the flat form.
std::vector<std::string> check_invariant(const otprg_cluster_state& st, const otprg_copy_instance& in) {
  std::vector<std::string> v;
  auto fail = [&](std::string m) { v.push_back(std::move(m)); };
  const int64_t bound = in.unit_ceil + 2;
  auto dem_count = [&](int32_t c) {
    int64_t t = st.dem_free[c];
    for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f) t += st.flow_cnt[f];
    return t;
  };
  for (int32_t a = 0; a < st.n_a; ++a) {
    std::vector<int64_t> values;
    int64_t total = 0;
    const std::string at = std::to_string(a);
    for (int32_t c = st.dem_off[a]; c < st.dem_off[a + 1]; ++c) {
      const int64_t cnt = dem_count(c), y = st.dem_y[c];
      if (cnt == 0) continue;
      values.push_back(y);
      total += cnt;
      if (y > 0) fail("demand cluster with positive dual at a=" + at);
      if (std::llabs(y) > bound) fail("demand cluster dual exceeds magnitude bound at a=" + at);
      if (st.dem_free[c] > 0 && y != 0) fail("free demand copies away from dual zero at a=" + at);
      for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f)
        if (st.flow_b[f] < 0 || st.flow_b[f] >= st.n_b || st.flow_cnt[f] <= 0)
          fail("bad flow entry at a=" + at);
    }
    std::sort(values.begin(), values.end());
    values.erase(std::unique(values.begin(), values.end()), values.end());
    if (values.size() > 2) fail("more than two distinct duals among copies of a=" + at);
    if (total != in.demand_copies[a]) fail("demand copy count mismatch at a=" + at);
  }
  for (int32_t b = 0; b < st.n_b; ++b) {
    std::vector<int64_t> values;
    int64_t total = 0, free_clusters = 0;
    int64_t max_y = std::numeric_limits<int64_t>::min();
    const std::string at = std::to_string(b);
    for (int32_t c = st.sup_off[b]; c < st.sup_off[b + 1]; ++c) {
      const int64_t cnt = st.sup_free[c] + st.sup_matched[c], y = st.sup_y[c];
      if (cnt == 0) continue;
      values.push_back(y);
      total += cnt;
      max_y = std::max(max_y, y);
      if (y < 0) fail("supply cluster with negative dual at b=" + at);
      if (std::llabs(y) > bound) fail("supply cluster dual exceeds magnitude bound at b=" + at);
      if (st.sup_free[c] > 0) ++free_clusters;
    }
    std::sort(values.begin(), values.end());
    values.erase(std::unique(values.begin(), values.end()), values.end());
    if (values.size() > 2) fail("more than two distinct duals among copies of b=" + at);
    if (total != in.supply_copies[b]) fail("supply copy count mismatch at b=" + at);
    if (free_clusters > 1) fail("free supply copies split across duals at b=" + at);
    for (int32_t c = st.sup_off[b]; c < st.sup_off[b + 1]; ++c)
      if (st.sup_free[c] + st.sup_matched[c] > 0 && st.sup_free[c] > 0 && st.sup_y[c] != max_y)
        fail("free supply copies below their vertex maximum dual at b=" + at);
  }
  std::vector<int64_t> inbound(st.n_b, 0);
  for (int32_t c = 0; c < st.dem_off[st.n_a]; ++c)
    for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f)
      if (st.flow_b[f] >= 0 && st.flow_b[f] < st.n_b) inbound[st.flow_b[f]] += st.flow_cnt[f];
  for (int32_t b = 0; b < st.n_b; ++b) {
    int64_t matched = 0;
    for (int32_t c = st.sup_off[b]; c < st.sup_off[b + 1]; ++c) matched += st.sup_matched[c];
    if (inbound[b] != matched)
      fail("flow into b=" + std::to_string(b) + " disagrees with matched supply count");
  }
  return v;
}

// check_cluster_feasibility (ot.cpp:267-315) on the flat form.
std::vector<std::string> check_feasibility(const otprg_cluster_state& st, const otprg_copy_instance& in) {
  std::vector<std::string> v;
  auto k = [&](int32_t a, int32_t b) { return static_cast<int64_t>(in.k[static_cast<size_t>(a) * in.n_b + b]); };
  // matched copy pairs are tight: expected[b][partner dual] from the flows
  std::vector<std::vector<std::pair<int64_t, int64_t>>> expected(st.n_b), actual(st.n_b);
  auto add = [](std::vector<std::pair<int64_t, int64_t>>& m, int64_t y, int64_t c) {
    for (auto& e : m)
      if (e.first == y) {
        e.second += c;
        return;
      }
    m.emplace_back(y, c);
  };
  for (int32_t a = 0; a < st.n_a; ++a)
    for (int32_t c = st.dem_off[a]; c < st.dem_off[a + 1]; ++c)
      for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f)
        add(expected[st.flow_b[f]], k(a, st.flow_b[f]) - st.dem_y[c], st.flow_cnt[f]);
  for (int32_t b = 0; b < st.n_b; ++b) {
    for (int32_t c = st.sup_off[b]; c < st.sup_off[b + 1]; ++c)
      if (st.sup_matched[c] > 0) add(actual[b], st.sup_y[c], st.sup_matched[c]);
    auto& e = expected[b];
    auto& x = actual[b];
    std::sort(e.begin(), e.end());
    std::sort(x.begin(), x.end());
    if (e != x) v.push_back("matched copies of b=" + std::to_string(b) + " are not tight against their partners");
  }
  // unmatched cross pairs respect the dual-sum allowance
  for (int32_t a = 0; a < st.n_a; ++a)
    for (int32_t c = st.dem_off[a]; c < st.dem_off[a + 1]; ++c) {
      int64_t cnt_a = st.dem_free[c];
      for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f) cnt_a += st.flow_cnt[f];
      if (cnt_a == 0) continue;
      const int64_t ya = st.dem_y[c];
      for (int32_t b = 0; b < st.n_b; ++b) {
        const int64_t kk = k(a, b);
        for (int32_t d = st.sup_off[b]; d < st.sup_off[b + 1]; ++d) {
          const int64_t cnt_b = st.sup_free[d] + st.sup_matched[d];
          if (cnt_b == 0) continue;
          int64_t cross = 0;
          if (kk - ya == st.sup_y[d])
            for (int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f)
              if (st.flow_b[f] == b) cross = st.flow_cnt[f];
          if (cnt_a * cnt_b > cross && ya + st.sup_y[d] > kk + 1)
            v.push_back("dual-sum allowance violated between copies of a=" + std::to_string(a) +
                        " and b=" + std::to_string(b));
        }
      }
    }
  return v;
}

class OtSolver {
 public:
  OtSolver(otprg_ctx* ctx, const otprg_ot_problem* p, otprg_ot_result* r,
           const otprg_ot_options* opt = nullptr)
      : ctx_(ctx), p_(p), r_(r), opt_(opt) {}

  void run() {
    Timer total;
    validate_ot(p_);
    if (!(p_->eps > 0.0 && p_->eps < 1.0)) throw OtError{OTPRG_PARAMETER, "eps must lie in (0, 1)"};
    eps_in_ = p_->eps / 3.0;  // ot.cpp:710
    sm_ = scale_and_round(p_, eps_in_);
    n_a_ = p_->n_a;
    n_b_ = p_->n_b;
    build_costs();
    if (debug()) {  // the CopyInstance the hooks see: k at eps/3 on the host
      hk_store_.resize(static_cast<size_t>(n_a_) * n_b_);
      for (size_t i = 0; i < hk_store_.size(); ++i)
        hk_store_[i] = static_cast<int32_t>(host_scaled_floor(p_->cost[i], eps_in_));
      hk_ = hk_store_.data();
    }
    solve_copy_matching();
    save_state();
    plan_from_flow();
    r_->theta = sm_.theta;
    r_->total_d = sm_.total_d;
    r_->total_s = sm_.total_s;
    r_->solve_ms = total.ms();
  }

  // solve_copy_matching on a given copy instance (ot.cpp:418-637).
  void run_copy(const otprg_copy_instance* ci, double eps, otprg_copy_result* cr) {
    if (!ci || !ci->k || !ci->demand_copies || !ci->supply_copies || ci->n_a < 0 || ci->n_b < 0)
      throw OtError{OTPRG_PARAMETER, "copy counts do not match the cost matrix"};
    int64_t td = 0, ts = 0;
    for (int32_t a = 0; a < ci->n_a; ++a) {
      if (ci->demand_copies[a] < 0) throw OtError{OTPRG_PARAMETER, "negative demand copy count"};
      td += ci->demand_copies[a];
    }
    for (int32_t b = 0; b < ci->n_b; ++b) {
      if (ci->supply_copies[b] < 0) throw OtError{OTPRG_PARAMETER, "negative supply copy count"};
      ts += ci->supply_copies[b];
    }
    if (ts > td) throw OtError{OTPRG_PARAMETER, "copy instance needs total supply <= total demand"};
    if (!(eps > 0.0 && eps < 1.0)) throw OtError{OTPRG_PARAMETER, "eps must lie in (0, 1)"};
    n_a_ = ci->n_a;
    n_b_ = ci->n_b;
    eps_in_ = eps;
    sm_.theta = 0.0;
    sm_.d.assign(ci->demand_copies, ci->demand_copies + n_a_);
    sm_.s.assign(ci->supply_copies, ci->supply_copies + n_b_);
    sm_.total_d = td;
    sm_.total_s = ts;
    hk_ = ci->k;
    unit_ceil_ = ci->unit_ceil;
    otprg_ot_result tmp{};
    tmp.free_counts = cr->free_counts;
    tmp.free_cap = cr->free_cap;
    r_ = &tmp;
    if (n_a_ > 0 && n_b_ > 0) {
      build_costs_from_k();
      solve_copy_matching();
    } else {  // nothing to match: the loop ends at once (n_i = 0)
      st_ = initial_state();
      flow_.assign(n_a_, {});
      tmp.full_match_termination = 1;
    }
    save_state();
    cr->phases = tmp.phases;
    cr->sum_ni = tmp.sum_ni;
    cr->full_match_termination = tmp.full_match_termination;
    cr->gpu_launches = tmp.gpu_launches;
    if (cr->flow) {
      std::memset(cr->flow, 0, static_cast<size_t>(n_a_) * n_b_ * 8);
      for (int32_t a = 0; a < n_a_; ++a)
        for (const auto& [b, f] : flow_[a]) cr->flow[static_cast<size_t>(a) * n_b_ + b] = f;
    }
  }

  // plan_from_flow alone on a dense flow (ot.cpp:639-703).
  void run_plan(const int64_t* flow, double theta) {
    if (!p_->mu || !p_->nu || !p_->cost || p_->n_a < 0 || p_->n_b < 0)
      throw OtError{OTPRG_PARAMETER, "flow matrix dimensions do not match the instance"};
    n_a_ = p_->n_a;
    n_b_ = p_->n_b;
    sm_.theta = theta;
    flow_.assign(n_a_, {});
    for (int32_t a = 0; a < n_a_; ++a)
      for (int32_t b = 0; b < n_b_; ++b) {
        const int64_t f = flow[static_cast<size_t>(a) * n_b_ + b];
        if (f < 0) throw OtError{OTPRG_PARAMETER, "negative flow entry"};
        if (f > 0) flow_[a].emplace_back(b, f);
      }
    plan_from_flow();
  }

 private:
  otprg_ctx* ctx_;
  const otprg_ot_problem* p_;
  otprg_ot_result* r_;
  const otprg_ot_options* opt_;
  double eps_in_ = 0.0;
  ScaledMasses sm_;
  int32_t n_a_ = 0, n_b_ = 0;
  int width_ = 2, lda_ = 0;
  int64_t unit_ceil_ = 0;                // dual bound - 2 of the hooks' CopyInstance
  const int32_t* hk_ = nullptr;          // host k (copy instance / debug mode), row-major
  std::vector<int32_t> hk_store_;
  FlatState st_;                         // ClusterState exported from the device (hooks, final)
  std::vector<std::vector<std::pair<int32_t, int64_t>>> flow_;  // final sparse flow per a

  bool debug() const { return opt_ && (opt_->check_invariants || opt_->observer); }


  otprg_copy_instance copy_instance() const {
    return otprg_copy_instance{n_a_, n_b_, hk_, unit_ceil_, sm_.d.data(), sm_.s.data()};
  }

  // ClusterSolveResult::state (before completion) kept on the context.
  void save_state() { ctx_->ot_state = std::make_shared<FlatState>(st_); }

  // The state solve_copy_matching starts from (ot.cpp:430-437): one demand
  // cluster at dual 0 with every copy free, one supply cluster at dual 1.
  FlatState initial_state() const {
    FlatState f;
    f.n_a = n_a_;
    f.n_b = n_b_;
    f.dem_off.assign(1, 0);
    f.flow_off.assign(1, 0);
    f.sup_off.assign(1, 0);
    for (int32_t a = 0; a < n_a_; ++a) {
      if (sm_.d[a] > 0) {
        f.dem_y.push_back(0);
        f.dem_free.push_back(sm_.d[a]);
        f.flow_off.push_back(0);
      }
      f.dem_off.push_back(static_cast<int32_t>(f.dem_y.size()));
    }
    for (int32_t b = 0; b < n_b_; ++b) {
      if (sm_.s[b] > 0) {
        f.sup_y.push_back(1);
        f.sup_free.push_back(sm_.s[b]);
        f.sup_matched.push_back(0);
      }
      f.sup_off.push_back(static_cast<int32_t>(f.sup_y.size()));
    }
    return f;
  }

  // scale_round_costs(costs, eps/3) on the device (core.cpp:34-53), kT[b][a].
  void build_costs() {
    Timer t;
    if (!(eps_in_ > 0.0 && eps_in_ < 1.0)) throw OtError{OTPRG_PARAMETER, "eps must lie in (0, 1)"};
    const int64_t uf = host_scaled_floor(1.0, eps_in_);
    if (uf + 4 > std::numeric_limits<int32_t>::max())
      throw OtError{OTPRG_PARAMETER, "eps too small: 1/eps overflows the cost unit type"};
    const int64_t uc = static_cast<double>(uf) * eps_in_ == 1.0 ? uf : uf + 1;
    unit_ceil_ = uc;
    width_ = otprg::storage_width(uc + 2, OTPRG_STORAGE_AUTO);
    if (width_ < 0) throw OtError{OTPRG_PARAMETER, "eps too small for the device cost storage"};
    const int align = 512 / width_;
    lda_ = (n_a_ + align - 1) / align * align;
    OT_CK(cudaSetDevice(ctx_->device), "cudaSetDevice");
    const size_t bytes = static_cast<size_t>(n_a_) * n_b_ * sizeof(double);
    ctx_->stage_holds_cost = false;
    OT_CK(ctx_->stage.ensure(bytes), "alloc cost staging");
    OT_CK(ctx_->kT.ensure(static_cast<size_t>(n_b_) * lda_ * width_), "alloc kT");
    OT_CK(ctx_->ctl.ensure(sizeof(otprg::Ctl)), "alloc ctl");
    OT_CK(otprg::h2d_large(ctx_, ctx_->stage.p, p_->cost, bytes), "H2D cost");
    OT_CK(cudaMemsetAsync(ctx_->ctl.p, 0, sizeof(otprg::Ctl), ctx_->stream), "memset");
    int* status = &ctx_->ctl.as<otprg::Ctl>()->status;
    OT_CK(otprg::launch_round_dense(ctx_->stage.as<double>(), n_a_, n_b_, false, eps_in_, ctx_->kT.p,
                                    lda_, width_, status, ctx_->stream),
          "round_dense launch");
    int dstatus = 0;
    OT_CK(cudaMemcpyAsync(&dstatus, status, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream),
          "D2H status");
    OT_CK(cudaStreamSynchronize(ctx_->stream), "cost build");
    if (dstatus) throw OtError{OTPRG_PARAMETER, "OT cost entry outside [0,1]"};
    launches_ += 1;
    r_->build_ms = t.ms();
    alloc_device();
  }

  // The copy instance's k (host int32, row-major) -> kT on the device.
  void build_costs_from_k() {
    Timer t;
    int64_t kmax = 0;
    const size_t nn = static_cast<size_t>(n_a_) * n_b_;
    for (size_t i = 0; i < nn; ++i) {
      if (hk_[i] < 0) throw OtError{OTPRG_PARAMETER, "negative rounded cost in the copy instance"};
      kmax = std::max<int64_t>(kmax, hk_[i]);
    }
    width_ = otprg::storage_width(std::max(kmax, unit_ceil_) + 2, OTPRG_STORAGE_AUTO);
    if (width_ < 0) throw OtError{OTPRG_PARAMETER, "rounded costs beyond the device cost storage"};
    const int align = 512 / width_;
    lda_ = (n_a_ + align - 1) / align * align;
    OT_CK(cudaSetDevice(ctx_->device), "cudaSetDevice");
    ctx_->stage_holds_cost = false;
    OT_CK(ctx_->stage.ensure(nn * 4), "alloc k staging");
    OT_CK(ctx_->kT.ensure(static_cast<size_t>(n_b_) * lda_ * width_), "alloc kT");
    OT_CK(ctx_->ctl.ensure(sizeof(otprg::Ctl)), "alloc ctl");
    OT_CK(otprg::h2d_large(ctx_, ctx_->stage.p, hk_, nn * 4), "H2D k");
    OT_CK(otprg::launch_k_to_kT(ctx_->stage.as<int32_t>(), n_a_, n_b_, ctx_->kT.p, lda_, width_, ctx_->stream),
          "k_to_kT launch");
    OT_CK(cudaStreamSynchronize(ctx_->stream), "k upload");
    launches_ += 1;
    r_->build_ms = t.ms();
    alloc_device();
  }

  // ---- device state (ot_device.cu) --------------------------------------------
  // ctx->ot_dev[] slots
  enum Buf {
    bT, bDy, bDfree, bDmatched, bConsumed, bFlOff, bFlCode, bFlB, bFlCnt, bFlPre, bSy, bSfree, bSmatched,
    bSfreed, bFb, bFy, bFpos, bFidx, bFu0, bFu, bAdmLen, bAdmOff, bAdm, bEk0, bEv0, bEk1, bEv1, bRk0, bRv0,
    bRk1, bRv1, bCtr, bTemp, bScratch, bCut, bDaCnt, bDaFill, bDaOff, bDaTouch, bBar, bLoop, bFcounts, bRecOff, bStep, bNum
  };
  otprg::OtDev D_{};
  int64_t fl_cap_ = 0, adm_cap_ = 0, e_cap_ = 0, r_cap_ = 0;
  size_t temp_cap_ = 0;
  int launches_ = 0;
  int64_t scan_bytes_ = 0;
  int64_t* hctr_ = nullptr;  // pinned: counters + status
  // DA rounds launched per host look (0: the sorted, one-sync-per-round path;
  // OTPRG_OT_DA_BATCH), rounds that fell back to the sort
  int da_batch_ = [] {
    const char* e = std::getenv("OTPRG_OT_DA_BATCH");
    return e ? std::max(0, std::atoi(e)) : 4;
  }();
  int64_t sorted_rounds_ = 0;

  DevBuf& buf(Buf b) { return ctx_->ot_dev[b]; }
  template <typename T>
  T* ensure(Buf b, size_t n) {
    OT_CK(buf(b).ensure(std::max<size_t>(n, 1) * sizeof(T)), "alloc OT device state");
    return buf(b).as<T>();
  }

  void alloc_device() {
    static_assert(bNum <= 48, "ot_dev slots");
    if (n_b_ >= (1 << 21) - 1 || n_a_ >= (1 << 21) || unit_ceil_ + 4 >= (1 << 19))
      throw OtError{OTPRG_PARAMETER, "OT instance beyond the device state's index range (n < 2^21, 1/eps < 2^19)"};
    const size_t na2 = 2 * static_cast<size_t>(n_a_), nb = n_b_, nb2 = 2 * nb;
    D_.n_a = n_a_;
    D_.n_b = n_b_;
    D_.lda = lda_;
    D_.width = width_;
    D_.kT = ctx_->kT.p;
    D_.t = ensure<char>(bT, 2 * static_cast<size_t>(lda_) * width_);
    D_.dy = ensure<int32_t>(bDy, na2);
    D_.dfree = ensure<int64_t>(bDfree, na2);
    D_.dmatched = ensure<int64_t>(bDmatched, na2);
    D_.consumed = ensure<int64_t>(bConsumed, na2);
    D_.cl_cut = ensure<int32_t>(bCut, na2);
    D_.fl_off = ensure<int64_t>(bFlOff, na2 + 1);
    D_.sy = ensure<int32_t>(bSy, nb2);
    D_.sfree = ensure<int64_t>(bSfree, nb2);
    D_.smatched = ensure<int64_t>(bSmatched, nb2);
    D_.sfreed = ensure<int64_t>(bSfreed, nb2);
    D_.fb = ensure<int32_t>(bFb, nb);
    D_.fy = ensure<int32_t>(bFy, nb);
    D_.fpos = ensure<int32_t>(bFpos, nb);
    D_.fidx = ensure<int32_t>(bFidx, nb);
    D_.fu0 = ensure<int64_t>(bFu0, nb);
    D_.fu = ensure<int64_t>(bFu, nb);
    D_.adm_len = ensure<int64_t>(bAdmLen, nb + 1);
    D_.adm_off = ensure<int64_t>(bAdmOff, nb + 1);
    D_.da_cnt = ensure<int32_t>(bDaCnt, na2);
    D_.da_fill = ensure<int32_t>(bDaFill, na2);
    D_.da_off = ensure<int64_t>(bDaOff, na2);
    D_.da_touch = ensure<int32_t>(bDaTouch, na2);
    OT_CK(cudaMemsetAsync(D_.da_cnt, 0, na2 * 4, ctx_->stream), "memset");
    OT_CK(cudaMemsetAsync(D_.da_fill, 0, na2 * 4, ctx_->stream), "memset");
    D_.ctr = ensure<int64_t>(bCtr, otprg::kCtrCount + 8);
    D_.status = reinterpret_cast<int*>(D_.ctr + otprg::kCtrCount);
    D_.err = reinterpret_cast<int32_t*>(D_.ctr + otprg::kCtrCount + 1);
    fl_cap_ = adm_cap_ = e_cap_ = r_cap_ = 0;
    grow_flows(na2);
    if (ctx_->ot_hpin_n < 256) {
      if (ctx_->ot_hpin) cudaFreeHost(ctx_->ot_hpin);
      ctx_->ot_hpin = nullptr;
      ctx_->ot_hpin_n = 0;
      OT_CK(cudaMallocHost(&ctx_->ot_hpin, 256), "pinned staging");
      ctx_->ot_hpin_n = 256;
    }
    hctr_ = static_cast<int64_t*>(ctx_->ot_hpin);
  }

  void grow_flows(int64_t n) {
    if (n <= fl_cap_) return;
    const int64_t c = std::max<int64_t>(n, fl_cap_ * 3 / 2);
    // (a growth keeps nothing: called before the rebuild writes the new flows)
    D_.fl_code = ensure<int32_t>(bFlCode, c);
    D_.fl_b = ensure<int32_t>(bFlB, c);
    D_.fl_cnt = ensure<int64_t>(bFlCnt, c);
    D_.fl_pre = ensure<int64_t>(bFlPre, c);
    fl_cap_ = c;
  }

  void grow(int64_t& cap, int64_t n, Buf k0, Buf v0, Buf k1, Buf v1, bool keep0) {
    if (n <= cap) return;
    const int64_t c = std::max<int64_t>(n, cap * 3 / 2);
    if (keep0 && cap > 0) {  // the live prefix of buffer 0 moves along
      DevBuf tk, tv;
      OT_CK(tk.ensure(cap * 8), "alloc");
      OT_CK(tv.ensure(cap * 8), "alloc");
      OT_CK(cudaMemcpyAsync(tk.p, buf(k0).p, cap * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(tv.p, buf(v0).p, cap * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      ensure<unsigned long long>(k0, c);
      ensure<int64_t>(v0, c);
      OT_CK(cudaMemcpyAsync(buf(k0).p, tk.p, cap * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(buf(v0).p, tv.p, cap * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaStreamSynchronize(ctx_->stream), "grow");
    } else {
      ensure<unsigned long long>(k0, c);
      ensure<int64_t>(v0, c);
    }
    ensure<unsigned long long>(k1, c);
    ensure<int64_t>(v1, c);
    cap = c;
  }

  void temp_need(size_t bytes) {
    if (bytes > temp_cap_) {
      ensure<char>(bTemp, bytes);
      temp_cap_ = bytes;
    }
  }
  void sort(const unsigned long long* kin, unsigned long long* kout, const int64_t* vin, int64_t* vout, int64_t n,
            int end_bit) {
    size_t tb = 0;
    OT_CK(otprg::ot_sort_pairs(nullptr, tb, kin, kout, vin, vout, n, end_bit, ctx_->stream), "sort size");
    temp_need(tb);
    tb = temp_cap_;
    OT_CK(otprg::ot_sort_pairs(buf(bTemp).p, tb, kin, kout, vin, vout, n, end_bit, ctx_->stream), "sort");
    launches_ += 4;
  }

  // Counters / status to the host (one sync).
  void read_ctr() {
    OT_CK(cudaMemcpyAsync(hctr_, D_.ctr, (otprg::kCtrCount + 5) * 8, cudaMemcpyDeviceToHost, ctx_->stream), "D2H");
    OT_CK(cudaStreamSynchronize(ctx_->stream), "OT phase");
    check_status();
  }
  void check_status() {
    const int* st = reinterpret_cast<const int*>(hctr_ + otprg::kCtrCount);
    const int32_t* err = reinterpret_cast<const int32_t*>(hctr_ + otprg::kCtrCount + 1);
    if (st[0] == 0) return;
    switch (err[0]) {
      case 1: throw OtError{OTPRG_INVARIANT, "third dual value among copies of demand vertex " + std::to_string(err[1])};
      case 2: throw OtError{OTPRG_INVARIANT, "third dual value among copies of supply vertex " + std::to_string(err[1])};
      case 3: throw OtError{OTPRG_INVARIANT, "displaced supply copy has no cluster"};
      case 4: throw OtError{OTPRG_INVARIANT, "demand dual beyond the device storage at a=" + std::to_string(err[1])};
      default: throw OtError{OTPRG_INVARIANT, "OT device state corrupt"};
    }
  }

  // Initial state (ot.cpp:430-437) to the device.
  void upload_initial() {
    const size_t na2 = 2 * static_cast<size_t>(n_a_), nb2 = 2 * static_cast<size_t>(n_b_);
    std::vector<int32_t> dy(na2, INT32_MIN), sy(nb2, INT32_MIN), code, fb;
    std::vector<int64_t> dfree(na2, 0), dz(na2, 0), sfree(nb2, 0), sz(nb2, 0), off(na2 + 1, 0), cnt, pre;
    for (int32_t a = 0; a < n_a_; ++a) {
      off[2 * a] = static_cast<int64_t>(code.size());
      if (sm_.d[a] > 0) {
        dy[2 * a] = 0;
        dfree[2 * a] = sm_.d[a];
        code.push_back(2 * a);
        fb.push_back(otprg::kFreeB);
        cnt.push_back(sm_.d[a]);
        pre.push_back(0);
      }
      off[2 * a + 1] = static_cast<int64_t>(code.size());
    }
    off[na2] = static_cast<int64_t>(code.size());
    for (int32_t b = 0; b < n_b_; ++b)
      if (sm_.s[b] > 0) {
        sy[2 * b] = 1;
        sfree[2 * b] = sm_.s[b];
      }
    grow_flows(static_cast<int64_t>(code.size()));
    cudaStream_t s = ctx_->stream;
    auto up = [&](void* d, const void* h, size_t bytes) {
      if (bytes) OT_CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "H2D OT state");
    };
    up(D_.dy, dy.data(), na2 * 4);
    up(D_.dfree, dfree.data(), na2 * 8);
    up(D_.dmatched, dz.data(), na2 * 8);
    up(D_.consumed, dz.data(), na2 * 8);
    up(D_.fl_off, off.data(), (na2 + 1) * 8);
    up(D_.fl_code, code.data(), code.size() * 4);
    up(D_.fl_b, fb.data(), fb.size() * 4);
    up(D_.fl_cnt, cnt.data(), cnt.size() * 8);
    up(D_.fl_pre, pre.data(), pre.size() * 8);
    up(D_.sy, sy.data(), nb2 * 4);
    up(D_.sfree, sfree.data(), nb2 * 8);
    up(D_.smatched, sz.data(), nb2 * 8);
    up(D_.sfreed, sz.data(), nb2 * 8);
    OT_CK(cudaMemsetAsync(D_.ctr, 0, (otprg::kCtrCount + 5) * 8, s), "memset");
    n_flows_ = static_cast<int64_t>(code.size());
  }
  int64_t n_flows_ = 0;

  // The device ClusterState as a flat host state (dem clusters in slot order).
  FlatState export_state() {
    const size_t na2 = 2 * static_cast<size_t>(n_a_), nb2 = 2 * static_cast<size_t>(n_b_);
    std::vector<int32_t> dy(na2), sy(nb2), fb(n_flows_);
    std::vector<int64_t> dfree(na2), dmatched(na2), off(na2 + 1), cnt(n_flows_), sfree(nb2), smatched(nb2);
    cudaStream_t s = ctx_->stream;
    auto down = [&](void* h, const void* d, size_t bytes) {
      if (bytes) OT_CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "D2H OT state");
    };
    down(dy.data(), D_.dy, na2 * 4);
    down(dfree.data(), D_.dfree, na2 * 8);
    down(dmatched.data(), D_.dmatched, na2 * 8);
    down(off.data(), D_.fl_off, (na2 + 1) * 8);
    down(fb.data(), D_.fl_b, n_flows_ * 4);
    down(cnt.data(), D_.fl_cnt, n_flows_ * 8);
    down(sy.data(), D_.sy, nb2 * 4);
    down(sfree.data(), D_.sfree, nb2 * 8);
    down(smatched.data(), D_.smatched, nb2 * 8);
    OT_CK(cudaStreamSynchronize(s), "OT state export");
    FlatState f;
    f.n_a = n_a_;
    f.n_b = n_b_;
    f.dem_off.assign(1, 0);
    f.flow_off.assign(1, 0);
    f.sup_off.assign(1, 0);
    for (int32_t a = 0; a < n_a_; ++a) {
      for (int sl = 0; sl < 2; ++sl) {
        const size_t c = 2 * static_cast<size_t>(a) + sl;
        if (dfree[c] + dmatched[c] == 0) continue;
        f.dem_y.push_back(dy[c]);
        f.dem_free.push_back(dfree[c]);
        for (int64_t e = off[c]; e < off[c + 1]; ++e)
          if (fb[e] != otprg::kFreeB) {
            f.flow_b.push_back(fb[e]);
            f.flow_cnt.push_back(cnt[e]);
          }
        f.flow_off.push_back(static_cast<int64_t>(f.flow_b.size()));
      }
      f.dem_off.push_back(static_cast<int32_t>(f.dem_y.size()));
    }
    for (int32_t b = 0; b < n_b_; ++b) {
      for (int sl = 0; sl < 2; ++sl) {
        const size_t c = 2 * static_cast<size_t>(b) + sl;
        if (sfree[c] + smatched[c] == 0) continue;
        f.sup_y.push_back(sy[c]);
        f.sup_free.push_back(sfree[c]);
        f.sup_matched.push_back(smatched[c]);
      }
      f.sup_off.push_back(static_cast<int32_t>(f.sup_y.size()));
    }
    return f;
  }

  // Greedy maximality (ot.cpp:524-533, check_invariants only): a supply vertex
  // left with free copies must have found every admissible cluster used up.
  void check_maximality(int32_t n_free) {
    std::vector<int64_t> len(n_free), off(n_free), fu(n_free), cons(2 * static_cast<size_t>(n_a_)),
        dfree(cons.size()), dmatched(cons.size());
    cudaStream_t s = ctx_->stream;
    OT_CK(cudaMemcpyAsync(len.data(), D_.adm_len, n_free * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(off.data(), D_.adm_off, n_free * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(fu.data(), D_.fu, n_free * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(cons.data(), D_.consumed, cons.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(dfree.data(), D_.dfree, cons.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(dmatched.data(), D_.dmatched, cons.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
    const int64_t total = n_free ? off[n_free - 1] + len[n_free - 1] : 0;
    std::vector<int32_t> adm(total);
    if (total) OT_CK(cudaMemcpyAsync(adm.data(), D_.adm, total * 4, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaStreamSynchronize(s), "maximality check");
    for (int32_t i = 0; i < n_free; ++i) {
      if (fu[i] == 0) continue;
      for (int64_t e = off[i]; e < off[i] + len[i]; ++e)
        if (dfree[adm[e]] + dmatched[adm[e]] - cons[adm[e]] > 0)
          throw OtError{OTPRG_INVARIANT, "greedy step left an admissible pair unmatched"};
    }
  }


  // The flow arrays grown with their live entries (n_flows_) kept.
  void grow_flows_keep(int64_t n) {
    if (n <= fl_cap_) return;
    const int64_t c = std::max<int64_t>(n, fl_cap_ * 3 / 2);
    const size_t live = static_cast<size_t>(n_flows_);
    DevBuf tmp;
    if (live) {
      OT_CK(tmp.ensure(live * 24), "alloc");
      char* t = static_cast<char*>(tmp.p);
      OT_CK(cudaMemcpyAsync(t, D_.fl_code, live * 4, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(t + live * 4, D_.fl_b, live * 4, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(t + live * 8, D_.fl_cnt, live * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(t + live * 16, D_.fl_pre, live * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaStreamSynchronize(ctx_->stream), "grow");
    }
    D_.fl_code = ensure<int32_t>(bFlCode, c);
    D_.fl_b = ensure<int32_t>(bFlB, c);
    D_.fl_cnt = ensure<int64_t>(bFlCnt, c);
    D_.fl_pre = ensure<int64_t>(bFlPre, c);
    fl_cap_ = c;
    if (live) {
      const char* t = static_cast<const char*>(tmp.p);
      OT_CK(cudaMemcpyAsync(D_.fl_code, t, live * 4, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(D_.fl_b, t + live * 4, live * 4, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(D_.fl_cnt, t + live * 8, live * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaMemcpyAsync(D_.fl_pre, t + live * 16, live * 8, cudaMemcpyDeviceToDevice, ctx_->stream), "copy");
      OT_CK(cudaStreamSynchronize(ctx_->stream), "grow");
    }
  }


  // solve_copy_matching as one cooperative launch for the whole phase loop
  // (ot_dev_phase_loop: the steps of the device-sized phase separated by grid
  // barriers, the claim rounds looped on the device); the host relaunches
  // only when the loop holds (capacity, a round for the sort, records beyond
  // one block's merge) after finishing that step, as in the launch-sequence
  // form below.
  void solve_copy_matching_persistent() {
    upload_initial();
    const double threshold = eps_in_ * static_cast<double>(sm_.total_s);
    const int64_t phase_cap =
        static_cast<int64_t>(std::ceil((1.0 + 2.0 * eps_in_) / (eps_in_ * eps_in_))) + 8;
    cudaStream_t s = ctx_->stream;
    int64_t holds = 0, relaunches = 0;
    std::vector<int64_t> free_counts;
    Timer loop_t;
    int* scratch = ensure<int>(bScratch, 256);
    const int end_bit = 21 + 1 + static_cast<int>(std::ceil(std::log2(2.0 * n_a_ + 1.0)));
    // (test knob: tiny buffers, so every hold of the loop is taken)
    const bool small_caps = std::getenv("OTPRG_OT_SMALL_CAPS") != nullptr;
    D_.bar = ensure<unsigned>(bBar, 2);
    D_.loop = ensure<int64_t>(bLoop, 4);
    D_.fc_cap = small_caps ? 3 : std::min<int64_t>(phase_cap + 2, int64_t(1) << 20);
    D_.fcounts = ensure<int64_t>(bFcounts, D_.fc_cap);
    D_.rec_off = ensure<int64_t>(bRecOff, static_cast<size_t>(n_a_) + 1);
    const bool steptime = std::getenv("OTPRG_OT_STEPTIME") != nullptr;
    D_.steptime = steptime ? ensure<unsigned long long>(bStep, 32) : nullptr;
    if (steptime) OT_CK(cudaMemsetAsync(D_.steptime, 0, 32 * 8, s), "memset");
    // (test knob: every record merge through the per-vertex buckets)
    // one-block bitonic merge up to 1,024 records, buckets beyond (scripts/ot_steptime.py:
    // n = 100 phases merge ~500 records, bitonic 12 us vs buckets 17 us per phase;
    // n = 1,000 ~4,000 records, bitonic 78 us vs buckets 27 us)
    D_.small_rec = std::getenv("OTPRG_OT_BUCKETS") ? 0 : 1024;
    OT_CK(cudaMemsetAsync(D_.bar, 0, 2 * sizeof(unsigned), s), "memset");
    OT_CK(cudaMemsetAsync(D_.loop, 0, 4 * sizeof(int64_t), s), "memset");
    if (adm_cap_ < 1 || small_caps) {
      adm_cap_ = small_caps ? 8 : std::max<int64_t>(int64_t(1) << 20, 8 * static_cast<int64_t>(n_b_));
      D_.adm = ensure<int32_t>(bAdm, adm_cap_);
    }
    D_.adm_cap = adm_cap_;
    auto set_caps = [&](int64_t n_flows) {
      if (small_caps) {  // (capacities exactly as needed now: the device checks hold the rest)
        e_cap_ = std::max<int64_t>(e_cap_, adm_cap_ + n_b_ + 1);
        ensure<unsigned long long>(bEk0, e_cap_);
        ensure<int64_t>(bEv0, e_cap_);
        ensure<unsigned long long>(bEk1, e_cap_);
        ensure<int64_t>(bEv1, e_cap_);
        D_.e_key = buf(bEk0).as<unsigned long long>();
        D_.e_val = buf(bEv0).as<int64_t>();
        D_.s_key = buf(bEk1).as<unsigned long long>();
        D_.s_val = buf(bEv1).as<int64_t>();
        D_.e_cap = e_cap_;
        const int64_t r = n_flows + 2 * static_cast<int64_t>(n_a_) + 17;
        grow(r_cap_, r, bRk0, bRv0, bRk1, bRv1, false);
        D_.r_key = buf(bRk0).as<unsigned long long>();
        D_.r_val = buf(bRv0).as<int64_t>();
        D_.r_key2 = buf(bRk1).as<unsigned long long>();
        D_.r_val2 = buf(bRv1).as<int64_t>();
        D_.r_cap = std::max<int64_t>(r, std::min<int64_t>(r_cap_, r));
        grow_flows_keep(r_cap_);
        return;
      }
      grow(e_cap_, adm_cap_ + n_b_ + 1, bEk0, bEv0, bEk1, bEv1, false);
      D_.e_key = buf(bEk0).as<unsigned long long>();
      D_.e_val = buf(bEv0).as<int64_t>();
      D_.s_key = buf(bEk1).as<unsigned long long>();
      D_.s_val = buf(bEv1).as<int64_t>();
      D_.e_cap = e_cap_;
      grow(r_cap_, 2 * n_flows + e_cap_ + 2 * static_cast<int64_t>(n_a_) + 16, bRk0, bRv0, bRk1, bRv1, false);
      D_.r_key = buf(bRk0).as<unsigned long long>();
      D_.r_val = buf(bRv0).as<int64_t>();
      D_.r_key2 = buf(bRk1).as<unsigned long long>();
      D_.r_val2 = buf(bRv1).as<int64_t>();
      D_.r_cap = r_cap_;
      grow_flows_keep(r_cap_);
    };
    auto read_loop = [&](int64_t* out, int n) {
      OT_CK(cudaMemcpyAsync(out, D_.loop, n * 8, cudaMemcpyDeviceToHost, s), "D2H");
      OT_CK(cudaStreamSynchronize(s), "OT loop counters");
    };
    auto drain = [&] {  // n_i of the phases of the launches so far
      int64_t lp[4];
      read_loop(lp, 4);
      if (lp[0] > 0) {
        const size_t k = free_counts.size();
        free_counts.resize(k + lp[0]);
        OT_CK(cudaMemcpyAsync(free_counts.data() + k, D_.fcounts, lp[0] * 8, cudaMemcpyDeviceToHost, s), "D2H");
        OT_CK(cudaStreamSynchronize(s), "free counts");
      }
      return lp[1];
    };
    // the live flow count of the device state (phases advance on the device):
    // the buffers' growth keeps that many entries
    auto device_flows = [&] {
      int64_t nfl = 0;
      OT_CK(cudaMemcpy(&nfl, D_.fl_off + 2 * static_cast<size_t>(n_a_), 8, cudaMemcpyDeviceToHost), "D2H");
      n_flows_ = nfl;
      return nfl;
    };
    set_caps(n_flows_);
    // the first phase's free list
    OT_CK(cudaMemsetAsync(D_.ctr, 0, otprg::kCtrCount * 8, s), "memset");
    OT_CK(otprg::ot_dev_free_list(D_, scratch, s), "free list");
    launches_ += 2;
    int stage = 0;
    int64_t rounds_total = 0;
    while (true) {
      const cudaError_t le = otprg::ot_dev_phase_loop(D_, stage, threshold, scratch, s);
      if (le != cudaSuccess && relaunches == 0 &&
          (le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorLaunchOutOfResources)) {
        // the loop's blocks are not co-resident here (e.g. other work holds the
        // SMs): nothing has changed yet, run the launch-sequence form instead
        cudaGetLastError();
        solve_copy_matching_dev();
        return;
      }
      OT_CK(le, "OT phase loop launch");
      ++relaunches;
      launches_ += 1;
      read_ctr();
      const int64_t hold = hctr_[otprg::kCtrHold];
      if (hold == 9) break;
      ++holds;
      if (hold == 10) {  // the free-count buffer is full: drain it
        rounds_total += drain();
        OT_CK(cudaMemsetAsync(D_.loop, 0, 4 * sizeof(int64_t), s), "memset");
        if (static_cast<int64_t>(free_counts.size()) > phase_cap)
          throw OtError{OTPRG_INVARIANT, "phase count exceeded the proven bound; solver state is corrupt"};
        stage = 0;
      } else if (hold == 1) {  // admissible lists / entries beyond their buffers
        const int64_t n_free = hctr_[otprg::kCtrFree];
        OT_CK(cudaMemcpyAsync(&hctr_[otprg::kCtrCount + 4], D_.adm_off + n_free, 8, cudaMemcpyDeviceToHost, s),
              "D2H");
        OT_CK(cudaStreamSynchronize(s), "admissible count");
        const int64_t total = hctr_[otprg::kCtrCount + 4];
        if (total > adm_cap_) {
          adm_cap_ = std::max<int64_t>(total + total / 4, adm_cap_ * 3 / 2);
          D_.adm = ensure<int32_t>(bAdm, adm_cap_);
          D_.adm_cap = adm_cap_;
        }
        set_caps(device_flows());
        stage = 1;
      } else if (hold == 2) {  // a claim round for the sort
        const int64_t n = hctr_[otprg::kCtrN];
        sort(buf(bEk0).as<unsigned long long>(), buf(bEk1).as<unsigned long long>(), buf(bEv0).as<int64_t>(),
             buf(bEv1).as<int64_t>(), n, std::min(64, end_bit));
        OT_CK(otprg::ot_dev_resolve(D_, buf(bEk1).as<unsigned long long>(), buf(bEv1).as<int64_t>(), n,
                                    buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), s),
              "resolve");
        OT_CK(otprg::ot_dev_da_clear(D_, s), "DA clear");
        OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrNew], 0, 8, s), "memset");
        OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrDone], 0, 8, s), "memset");
        OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrBig], 0, 8, s), "memset");
        launches_ += 2;
        ++sorted_rounds_;
        stage = 2;
      } else if (hold == 3) {  // records beyond one block: CUB sort + merge
        const int64_t n_rec = hctr_[otprg::kCtrRec];
        auto rk0 = buf(bRk0).as<unsigned long long>();
        auto rv0 = buf(bRv0).as<int64_t>();
        sort(rk0, buf(bRk1).as<unsigned long long>(), rv0, buf(bRv1).as<int64_t>(), n_rec, 63);
        long long* d_nu = reinterpret_cast<long long*>(&D_.ctr[otprg::kCtrNFlows]);
        size_t tb = 0;
        OT_CK(otprg::ot_reduce_by_key(nullptr, tb, buf(bRk1).as<unsigned long long>(), rk0, buf(bRv1).as<int64_t>(),
                                      rv0, d_nu, n_rec, s),
              "reduce size");
        temp_need(tb);
        tb = temp_cap_;
        OT_CK(otprg::ot_reduce_by_key(buf(bTemp).p, tb, buf(bRk1).as<unsigned long long>(), rk0,
                                      buf(bRv1).as<int64_t>(), rv0, d_nu, n_rec, s),
              "reduce");
        launches_ += 2;
        stage = 4;
      } else if (hold == 4) {  // records beyond r_cap: the flows of this phase decide
        const int64_t nfl = device_flows();
        set_caps(nfl + hctr_[otprg::kCtrE]);
        stage = 3;
      } else {
        throw OtError{OTPRG_INVARIANT, "OT device phase loop stopped in an unknown state"};
      }
      OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrHold], 0, 8, s), "memset");
    }
    rounds_total += drain();
    const int64_t phases = static_cast<int64_t>(free_counts.size());
    if (phases > phase_cap)
      throw OtError{OTPRG_INVARIANT, "phase count exceeded the proven bound; solver state is corrupt"};
    int64_t sum_ni = 0;
    for (int64_t v : free_counts) sum_ni += v;
    r_->full_match_termination = (hctr_[otprg::kCtrNi] == 0);
    if (phases > 0) n_flows_ = hctr_[otprg::kCtrNFlows];
    r_->phases = phases;
    r_->sum_ni = sum_ni;
    if (r_->free_counts && r_->free_cap > 0)
      std::memcpy(r_->free_counts, free_counts.data(),
                  static_cast<size_t>(std::min<int64_t>(phases, r_->free_cap)) * 8);
    st_ = export_state();
    r_->loop_ms = loop_t.ms();
    if (D_.steptime) {
      unsigned long long st[32];
      OT_CK(cudaMemcpy(st, D_.steptime, sizeof(st), cudaMemcpyDeviceToHost), "D2H");
      std::fprintf(stderr, "ot step times (us, summed):");
      for (int k = 1; k < 32; ++k)
        if (st[k]) std::fprintf(stderr, " %d:%.0f", k, st[k] * 1e-3);
      std::fprintf(stderr, "\n");
    }
    if (std::getenv("OTPRG_OT_PROFILE"))
      std::fprintf(stderr,
                   "ot loop %.2f ms: %lld phases, %lld DA rounds (%lld sorted), %lld holds (persistent, %lld launches)\n",
                   r_->loop_ms, (long long)phases, (long long)rounds_total, (long long)sorted_rounds_,
                   (long long)holds, (long long)relaunches);
    r_->scan_ms = 0.0;
    r_->bytes_touched = 0;
    r_->gpu_launches = launches_;
    complete();
  }

  // solve_copy_matching with device-sized phases: one phase is one launch
  // sequence (admissible lists, claim rounds, updates, record merge, CSR
  // rebuild, the next phase's free list) and one look at the counters; the
  // host steps in only when the phase holds (kCtrHold: admissible lists past
  // their capacity, claim rounds not over after the batch, more records than
  // one block merges), finishes that step and resumes the sequence there.
  // Capacities are grown before the phase from host-known bounds (entries <=
  // admissible + free, records <= flows + entries + 2 n_a).
  void solve_copy_matching_dev() {
    upload_initial();
    const double threshold = eps_in_ * static_cast<double>(sm_.total_s);
    const int64_t phase_cap =
        static_cast<int64_t>(std::ceil((1.0 + 2.0 * eps_in_) / (eps_in_ * eps_in_))) + 8;
    cudaStream_t s = ctx_->stream;
    int64_t phases = 0, sum_ni = 0, rounds_total = 0, holds = 0;
    std::vector<int64_t> free_counts;
    Timer loop_t;
    int* scratch = ensure<int>(bScratch, 256);
    const int end_bit = 21 + 1 + static_cast<int>(std::ceil(std::log2(2.0 * n_a_ + 1.0)));
    if (adm_cap_ < 1) {
      adm_cap_ = std::max<int64_t>(int64_t(1) << 20, 8 * static_cast<int64_t>(n_b_));
      D_.adm = ensure<int32_t>(bAdm, adm_cap_);
    }
    D_.adm_cap = adm_cap_;
    auto set_caps = [&](int64_t n_free) {
      grow(e_cap_, adm_cap_ + n_free + 1, bEk0, bEv0, bEk1, bEv1, false);
      D_.e_key = buf(bEk0).as<unsigned long long>();
      D_.e_val = buf(bEv0).as<int64_t>();
      D_.s_key = buf(bEk1).as<unsigned long long>();
      D_.s_val = buf(bEv1).as<int64_t>();
      grow(r_cap_, n_flows_ + e_cap_ + 2 * static_cast<int64_t>(n_a_) + 16, bRk0, bRv0, bRk1, bRv1, false);
      D_.r_key = buf(bRk0).as<unsigned long long>();
      D_.r_val = buf(bRv0).as<int64_t>();
      grow_flows_keep(r_cap_);
    };
    auto rk0 = [&] { return buf(bRk0).as<unsigned long long>(); };
    auto rv0 = [&] { return buf(bRv0).as<int64_t>(); };
    // stage 0: the phase from its start; 1 from the admissible fill; 2 from
    // the claim rounds; 3 from the CSR rebuild
    auto launch_from = [&](int stage) {
      if (stage <= 0) {
        OT_CK(otprg::ot_dev_phase_begin(D_, s), "memset");
        OT_CK(otprg::ot_dev_t(D_, s), "cluster duals");
        OT_CK(otprg::ot_dev_adm(D_, 0, s), "admissible count");
        OT_CK(otprg::ot_dev_adm_scan(D_, s), "admissible offsets");
        launches_ += 3;
      }
      if (stage <= 1) {
        OT_CK(otprg::ot_dev_adm(D_, 1, s), "admissible fill");
        OT_CK(otprg::ot_dev_cut_init(D_, s), "cut init");
        launches_ += 2;
      }
      if (stage <= 2) {
        OT_CK(otprg::ot_dev_da_rounds(D_, da_batch_, s), "DA rounds");
        OT_CK(otprg::ot_dev_da_gate(D_, s), "DA gate");
        OT_CK(otprg::ot_dev_consumed(D_, D_.e_key, D_.e_val, -1, s), "consumed");
        OT_CK(otprg::ot_dev_records(D_, D_.e_key, D_.e_val, -1, s), "records");
        OT_CK(otprg::ot_dev_small_merge(D_, rk0(), rv0(), s), "record merge");
        launches_ += 5 * da_batch_ + 6;
      }
      OT_CK(otprg::ot_dev_rebuild(D_, rk0(), rv0(), -1, s), "rebuild");
      OT_CK(cudaMemsetAsync(D_.ctr, 0, 8, s), "memset");  // n_i of the next phase
      OT_CK(otprg::ot_dev_free_list(D_, scratch, s), "free list");
      launches_ += 4;
    };
    auto clear_hold = [&] { OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrHold], 0, 8, s), "memset"); };
    // the first phase's free list
    OT_CK(cudaMemsetAsync(D_.ctr, 0, otprg::kCtrCount * 8, s), "memset");
    OT_CK(otprg::ot_dev_free_list(D_, scratch, s), "free list");
    launches_ += 2;
    read_ctr();
    while (true) {
      const int64_t n_i = hctr_[otprg::kCtrNi];
      const int32_t n_free = static_cast<int32_t>(hctr_[otprg::kCtrFree]);
      if (static_cast<double>(n_i) <= threshold) {
        r_->full_match_termination = (n_i == 0);
        break;
      }
      set_caps(n_free);
      scan_bytes_ += 2 * static_cast<int64_t>(n_free) * lda_ * width_;
      int stage = 0;
      while (true) {
        launch_from(stage);
        read_ctr();
        const int64_t hold = hctr_[otprg::kCtrHold];
        if (hold == 0) break;
        ++holds;
        if (hold == 1) {  // admissible lists beyond adm_cap: grow, refill
          int64_t total = 0;
          OT_CK(cudaMemcpyAsync(&hctr_[otprg::kCtrCount + 4], D_.adm_off + n_free, 8, cudaMemcpyDeviceToHost, s),
                "D2H");
          OT_CK(cudaStreamSynchronize(s), "admissible count");
          total = hctr_[otprg::kCtrCount + 4];
          adm_cap_ = std::max<int64_t>(total + total / 4, adm_cap_ * 3 / 2);
          D_.adm = ensure<int32_t>(bAdm, adm_cap_);
          D_.adm_cap = adm_cap_;
          set_caps(n_free);
          stage = 1;
        } else if (hold == 2) {  // claim rounds not over (or a round for the sort)
          if (hctr_[otprg::kCtrDone] == 2) {
            const int64_t n = hctr_[otprg::kCtrN];
            sort(buf(bEk0).as<unsigned long long>(), buf(bEk1).as<unsigned long long>(), buf(bEv0).as<int64_t>(),
                 buf(bEv1).as<int64_t>(), n, std::min(64, end_bit));
            OT_CK(otprg::ot_dev_resolve(D_, buf(bEk1).as<unsigned long long>(), buf(bEv1).as<int64_t>(), n,
                                        buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), s),
                  "resolve");
            OT_CK(otprg::ot_dev_da_clear(D_, s), "DA clear");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrNew], 0, 8, s), "memset");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrDone], 0, 8, s), "memset");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrBig], 0, 8, s), "memset");
            launches_ += 2;
            ++sorted_rounds_;
          }
          stage = 2;
        } else if (hold == 3) {  // records beyond one block: CUB sort + merge
          const int64_t n_rec = hctr_[otprg::kCtrRec];
          sort(rk0(), buf(bRk1).as<unsigned long long>(), rv0(), buf(bRv1).as<int64_t>(), n_rec, 63);
          long long* d_nu = reinterpret_cast<long long*>(&D_.ctr[otprg::kCtrNFlows]);
          size_t tb = 0;
          OT_CK(otprg::ot_reduce_by_key(nullptr, tb, buf(bRk1).as<unsigned long long>(), rk0(),
                                        buf(bRv1).as<int64_t>(), rv0(), d_nu, n_rec, s),
                "reduce size");
          temp_need(tb);
          tb = temp_cap_;
          OT_CK(otprg::ot_reduce_by_key(buf(bTemp).p, tb, buf(bRk1).as<unsigned long long>(), rk0(),
                                        buf(bRv1).as<int64_t>(), rv0(), d_nu, n_rec, s),
                "reduce");
          launches_ += 2;
          stage = 3;
        } else {
          throw OtError{OTPRG_INVARIANT, "OT device phase stopped in an unknown state"};
        }
        clear_hold();
      }
      n_flows_ = hctr_[otprg::kCtrNFlows];
      rounds_total += hctr_[otprg::kCtrRounds];
      phases += 1;
      free_counts.push_back(n_i);
      sum_ni += n_i;
      if (phases > phase_cap)
        throw OtError{OTPRG_INVARIANT, "phase count exceeded the proven bound; solver state is corrupt"};
    }
    r_->phases = phases;
    r_->sum_ni = sum_ni;
    if (r_->free_counts && r_->free_cap > 0)
      std::memcpy(r_->free_counts, free_counts.data(),
                  static_cast<size_t>(std::min<int64_t>(phases, r_->free_cap)) * 8);
    st_ = export_state();
    r_->loop_ms = loop_t.ms();
    if (std::getenv("OTPRG_OT_PROFILE"))
      std::fprintf(stderr, "ot loop %.2f ms: %lld phases, %lld DA rounds (%lld sorted), %lld holds (device-sized)\n",
                   r_->loop_ms, (long long)phases, (long long)rounds_total, (long long)sorted_rounds_,
                   (long long)holds);
    r_->scan_ms = 0.0;
    r_->bytes_touched = scan_bytes_;
    r_->gpu_launches = launches_;
    complete();
  }

  // solve_copy_matching (ot.cpp:418-637): the phases on the device.
  void solve_copy_matching() {
    if (!debug() && da_batch_ > 0 && !std::getenv("OTPRG_OT_HOST_SIZED")) {
      if (std::getenv("OTPRG_OT_SEQ")) solve_copy_matching_dev();
      else solve_copy_matching_persistent();
      return;
    }
    upload_initial();
    const double threshold = eps_in_ * static_cast<double>(sm_.total_s);
    const int64_t phase_cap =
        static_cast<int64_t>(std::ceil((1.0 + 2.0 * eps_in_) / (eps_in_ * eps_in_))) + 8;
    cudaStream_t s = ctx_->stream;
    int64_t phases = 0, sum_ni = 0, rounds_total = 0;
    std::vector<int64_t> free_counts;
    Timer loop_t;
    int* scratch = ensure<int>(bScratch, 256);
    if (debug()) st_ = export_state();
    while (true) {
      // free list + n_i (one sync: the termination test, ot.cpp:442-446)
      OT_CK(cudaMemsetAsync(D_.ctr, 0, otprg::kCtrCount * 8, s), "memset");
      OT_CK(otprg::ot_dev_free_list(D_, scratch, s), "free list");
      launches_ += 2;
      read_ctr();
      const int64_t n_i = hctr_[otprg::kCtrNi];
      const int32_t n_free = static_cast<int32_t>(hctr_[otprg::kCtrFree]);
      if (static_cast<double>(n_i) <= threshold) {
        r_->full_match_termination = (n_i == 0);
        break;
      }
      const int64_t sum_before = opt_ && opt_->observer ? st_.sum_abs_duals() : 0;
      // admissible clusters of every free b: count, offsets, fill
      OT_CK(otprg::ot_dev_t(D_, s), "cluster duals");
      OT_CK(otprg::ot_dev_adm(D_, 0, s), "admissible count");
      OT_CK(cudaMemsetAsync(D_.adm_len + n_free, 0, 8, s), "memset");
      {
        size_t tb = 0;
        OT_CK(otprg::ot_exclusive_sum(nullptr, tb, D_.adm_len, D_.adm_off, n_free + 1, s), "scan size");
        temp_need(tb);
        tb = temp_cap_;
        OT_CK(otprg::ot_exclusive_sum(buf(bTemp).p, tb, D_.adm_len, D_.adm_off, n_free + 1, s), "scan");
      }
      int64_t adm_total = 0;
      OT_CK(cudaMemcpyAsync(&hctr_[otprg::kCtrCount + 4], D_.adm_off + n_free, 8, cudaMemcpyDeviceToHost, s), "D2H");
      OT_CK(cudaStreamSynchronize(s), "admissible count");
      adm_total = hctr_[otprg::kCtrCount + 4];
      if (adm_total > adm_cap_) {
        adm_cap_ = std::max<int64_t>(adm_total, adm_cap_ * 3 / 2);
        D_.adm = ensure<int32_t>(bAdm, adm_cap_);
      }
      OT_CK(otprg::ot_dev_adm(D_, 1, s), "admissible fill");
      launches_ += 5;
      scan_bytes_ += 2 * static_cast<int64_t>(n_free) * lda_ * width_;
      // claims (K10): deferred-acceptance rounds; entries live in buffers 0
      grow(e_cap_, std::max<int64_t>(adm_total + n_free, 1), bEk0, bEv0, bEk1, bEv1, false);
      D_.e_key = buf(bEk0).as<unsigned long long>();
      D_.e_val = buf(bEv0).as<int64_t>();
      int64_t n_e = 0;
      const int end_bit = 21 + 1 + static_cast<int>(std::ceil(std::log2(2.0 * n_a_ + 1.0)));
      OT_CK(otprg::ot_dev_cut_init(D_, s), "cut init");
      launches_ += 1;
      D_.s_key = buf(bEk1).as<unsigned long long>();
      D_.s_val = buf(bEv1).as<int64_t>();
      if (da_batch_ > 0) {
        // device-sized rounds, da_batch_ per host look (ot_dev_da_rounds)
        while (true) {
          OT_CK(otprg::ot_dev_da_rounds(D_, da_batch_, s), "DA rounds");
          launches_ += 5 * da_batch_;
          read_ctr();
          const int64_t done = hctr_[otprg::kCtrDone];
          if (done == 1) break;
          if (done == 2) {  // a cluster with more entries than a warp resolves: this round sorted
            const int64_t n = hctr_[otprg::kCtrN];
            sort(buf(bEk0).as<unsigned long long>(), buf(bEk1).as<unsigned long long>(), buf(bEv0).as<int64_t>(),
                 buf(bEv1).as<int64_t>(), n, std::min(64, end_bit));
            OT_CK(otprg::ot_dev_resolve(D_, buf(bEk1).as<unsigned long long>(), buf(bEv1).as<int64_t>(), n,
                                        buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), s),
                  "resolve");
            OT_CK(otprg::ot_dev_da_clear(D_, s), "DA clear");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrNew], 0, 8, s), "memset");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrDone], 0, 8, s), "memset");
            OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrBig], 0, 8, s), "memset");
            launches_ += 2;
            ++sorted_rounds_;
          }
        }
        n_e = hctr_[otprg::kCtrE];
        rounds_total += hctr_[otprg::kCtrRounds];
      } else {
        while (true) {
          OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrNew], 0, 8, s), "memset");
          OT_CK(otprg::ot_dev_propose(D_, s), "propose");
          read_ctr();
          const int64_t n_new = hctr_[otprg::kCtrNew];
          n_e = hctr_[otprg::kCtrE];
          if (n_new == 0) break;
          const int64_t n = n_e + n_new;
          sort(buf(bEk0).as<unsigned long long>(), buf(bEk1).as<unsigned long long>(), buf(bEv0).as<int64_t>(),
               buf(bEv1).as<int64_t>(), n, std::min(64, end_bit));
          OT_CK(cudaMemsetAsync(&D_.ctr[otprg::kCtrE], 0, 8, s), "memset");
          OT_CK(otprg::ot_dev_resolve(D_, buf(bEk1).as<unsigned long long>(), buf(bEv1).as<int64_t>(), n,
                                      buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), s),
                "resolve");
          launches_ += 2;
          ++rounds_total;
        }
      }
      // updates (K11): consumed copies, displaced partners, records of the next state
      const int64_t rec_need = n_flows_ + n_e + 2 * static_cast<int64_t>(n_a_) + 16;
      grow(r_cap_, rec_need, bRk0, bRv0, bRk1, bRv1, false);
      D_.r_key = buf(bRk0).as<unsigned long long>();
      D_.r_val = buf(bRv0).as<int64_t>();
      if (opt_ && opt_->check_invariants) {
        OT_CK(otprg::ot_dev_consumed(D_, buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), n_e, s),
              "consumed");
        check_maximality(n_free);
      } else {
        OT_CK(otprg::ot_dev_consumed(D_, buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), n_e, s),
              "consumed");
      }
      OT_CK(otprg::ot_dev_records(D_, buf(bEk0).as<unsigned long long>(), buf(bEv0).as<int64_t>(), n_e, s),
            "records");
      launches_ += 4;
      read_ctr();
      const int64_t n_rec = hctr_[otprg::kCtrRec];
      sort(buf(bRk0).as<unsigned long long>(), buf(bRk1).as<unsigned long long>(), buf(bRv0).as<int64_t>(),
           buf(bRv1).as<int64_t>(), n_rec, 63);
      {
        long long* d_nu = reinterpret_cast<long long*>(&D_.ctr[otprg::kCtrCount + 4]);
        size_t tb = 0;
        OT_CK(otprg::ot_reduce_by_key(nullptr, tb, buf(bRk1).as<unsigned long long>(),
                                      buf(bRk0).as<unsigned long long>(), buf(bRv1).as<int64_t>(),
                                      buf(bRv0).as<int64_t>(), d_nu, n_rec, s),
              "reduce size");
        temp_need(tb);
        tb = temp_cap_;
        OT_CK(otprg::ot_reduce_by_key(buf(bTemp).p, tb, buf(bRk1).as<unsigned long long>(),
                                      buf(bRk0).as<unsigned long long>(), buf(bRv1).as<int64_t>(),
                                      buf(bRv0).as<int64_t>(), d_nu, n_rec, s),
              "reduce");
      }
      read_ctr();
      n_flows_ = hctr_[otprg::kCtrCount + 4];
      grow_flows(n_flows_);
      OT_CK(otprg::ot_dev_rebuild(D_, buf(bRk0).as<unsigned long long>(), buf(bRv0).as<int64_t>(), n_flows_, s),
            "rebuild");
      launches_ += 4;
      phases += 1;
      free_counts.push_back(n_i);
      sum_ni += n_i;
      if (debug()) {
        read_ctr();  // the rebuild's normalisation checks
        st_ = export_state();
        phase_hooks(phases, n_i, sum_before);
      }
      if (phases > phase_cap)
        throw OtError{OTPRG_INVARIANT, "phase count exceeded the proven bound; solver state is corrupt"};
    }
    r_->phases = phases;
    r_->sum_ni = sum_ni;
    if (r_->free_counts && r_->free_cap > 0)
      std::memcpy(r_->free_counts, free_counts.data(),
                  static_cast<size_t>(std::min<int64_t>(phases, r_->free_cap)) * 8);
    st_ = export_state();
    r_->loop_ms = loop_t.ms();
    if (std::getenv("OTPRG_OT_PROFILE"))
      std::fprintf(stderr, "ot loop %.2f ms: %lld phases, %lld DA rounds (%lld sorted)\n", r_->loop_ms,
                   (long long)phases, (long long)rounds_total, (long long)sorted_rounds_);
    r_->scan_ms = 0.0;
    r_->bytes_touched = scan_bytes_;
    r_->gpu_launches = launches_;
    complete();
  }

  // Flow matrix (sparse, per a ascending b) + completion (ot.cpp:615-635): the
  // leftover free supply copies go to spare demand copies, both ascending.
  void complete() {
    const FlatState& f = st_;
    flow_.assign(n_a_, {});
    std::vector<int64_t> spare(n_a_, 0);
    for (int32_t a = 0; a < n_a_; ++a) {
      auto& row = flow_[a];
      for (int32_t c = f.dem_off[a]; c < f.dem_off[a + 1]; ++c) {
        spare[a] += f.dem_free[c];
        for (int64_t e = f.flow_off[c]; e < f.flow_off[c + 1]; ++e) row.emplace_back(f.flow_b[e], f.flow_cnt[e]);
      }
      // (two clusters: merge their b-ascending lists)
      std::sort(row.begin(), row.end());
      size_t w = 0;
      for (size_t r = 0; r < row.size(); ++r) {
        if (w > 0 && row[w - 1].first == row[r].first) row[w - 1].second += row[r].second;
        else row[w++] = row[r];
      }
      row.resize(w);
    }
    int32_t a_cursor = 0;
    int64_t a_spare = n_a_ > 0 ? spare[0] : 0;
    for (int32_t b = 0; b < n_b_; ++b) {
      int64_t need = 0;
      for (int32_t c = f.sup_off[b]; c < f.sup_off[b + 1]; ++c) need += f.sup_free[c];
      while (need > 0) {
        while (a_spare == 0) {
          ++a_cursor;
          if (a_cursor >= n_a_) throw OtError{OTPRG_INVARIANT, "completion ran out of demand copies"};
          a_spare = spare[a_cursor];
        }
        const int64_t take = std::min(need, a_spare);
        auto& row = flow_[a_cursor];
        auto it = std::lower_bound(row.begin(), row.end(), std::make_pair(b, int64_t{0}));
        if (it != row.end() && it->first == b) it->second += take;
        else row.insert(it, {b, take});
        need -= take;
        a_spare -= take;
      }
    }
  }

  // check_invariants / observer after a phase (ot.cpp:594-608).
  void phase_hooks(int64_t phase, int64_t n_i, int64_t sum_before) {
    const otprg_cluster_state st = st_.view();
    const otprg_copy_instance in = copy_instance();
    if (opt_->check_invariants) {
      for (int which = 0; which < 2; ++which) {
        const auto v = which == 0 ? check_invariant(st, in) : check_feasibility(st, in);
        if (!v.empty()) throw OtError{OTPRG_INVARIANT, "phase " + std::to_string(phase) + ": " + v.front()};
      }
    }
    if (opt_->observer) {
      const otprg_cluster_snapshot snap{phase, n_i, sum_before, st_.sum_abs_duals(), in, st};
      if (opt_->observer(&snap, opt_->user) != 0)
        throw OtError{OTPRG_ABORTED, "observer stopped the solve at phase " + std::to_string(phase)};
    }
  }

  // plan_from_flow (ot.cpp:639-703) on the nonzero entries, reference order.
  void plan_from_flow() {
    const double* mu = p_->mu;
    const double* nu = p_->nu;
    std::vector<std::vector<std::pair<int32_t, double>>> sigma(n_a_);
    std::vector<double> row_mass(n_a_, 0.0), col_mass(n_b_, 0.0);
    for (int32_t a = 0; a < n_a_; ++a) {
      for (const auto& [b, f] : flow_[a]) {
        if (f < 0) throw OtError{OTPRG_PARAMETER, "negative flow entry"};
        if (f == 0) continue;
        const double m = static_cast<double>(f) / sm_.theta;
        sigma[a].emplace_back(b, m);
        row_mass[a] += m;
        col_mass[b] += m;
      }
    }
    std::vector<double> pool(n_b_, 0.0);
    for (int32_t b = 0; b < n_b_; ++b) pool[b] = std::max(0.0, nu[b] - col_mass[b]);
    for (int32_t a = 0; a < n_a_; ++a) {
      double excess = row_mass[a] - mu[a];
      if (excess <= 0.0) continue;
      for (auto& [b, s] : sigma[a]) {
        if (!(excess > 0.0)) break;
        if (s <= 0.0) continue;
        const double take = std::min(s, excess);
        s -= take;
        pool[b] += take;
        excess -= take;
        row_mass[a] -= take;
      }
    }
    // Ship each pool to demands with spare capacity, ascending a.  The
    // reference rescans a = 0.. for every b; capacities only shrink here, so
    // a vertex whose capacity is gone is unlinked from an ascending list and
    // the visit order (hence every addition) is unchanged.
    std::vector<int32_t> nxt(n_a_, -1);
    int32_t head = -1, tail = -1;
    for (int32_t a = 0; a < n_a_; ++a) {
      if (!(mu[a] - row_mass[a] > 0.0)) continue;
      if (tail < 0) head = a;
      else nxt[tail] = a;
      tail = a;
    }
    for (int32_t b = 0; b < n_b_; ++b) {
      double rest = pool[b];
      int32_t prev = -1, a = head;
      while (a >= 0 && rest > 0.0) {
        const double cap = mu[a] - row_mass[a];
        if (cap <= 0.0) {  // never positive again: unlink
          const int32_t n = nxt[a];
          if (prev < 0) head = n;
          else nxt[prev] = n;
          a = n;
          continue;
        }
        const double add = std::min(cap, rest);
        auto& row = sigma[a];
        auto it = std::lower_bound(row.begin(), row.end(), b,
                                   [](const std::pair<int32_t, double>& e, int32_t k) { return e.first < k; });
        if (it != row.end() && it->first == b) it->second += add;
        else row.insert(it, {b, add});
        row_mass[a] += add;
        rest -= add;
        prev = a;
        a = nxt[a];
      }
      if (rest > kMassTolerance)
        throw OtError{OTPRG_INVARIANT, "residual supply could not be placed"};
    }
    // entries row-major with sigma > 0, cost summed in that order
    int64_t ne = 0;
    double cost = 0.0;
    for (int32_t a = 0; a < n_a_; ++a)
      for (const auto& [b, s] : sigma[a]) {
        if (!(s > 0.0)) continue;
        if (ne < r_->entry_cap) {
          r_->ent_a[ne] = a;
          r_->ent_b[ne] = b;
          r_->ent_mass[ne] = s;
        }
        ++ne;
        cost += s * p_->cost[static_cast<size_t>(a) * n_b_ + b];
      }
    r_->n_entries = ne;
    r_->cost = cost;
  }
};

// ---- Sinkhorn baseline (sinkhorn.cpp:69-151, round_to_marginals :12-66) -----
void run_sinkhorn(otprg_ctx* ctx, const otprg_ot_problem* p, const otprg_sinkhorn_config* cfg,
                  otprg_sinkhorn_result* r) {
  validate_ot(p);
  if (!cfg || !(cfg->reg > 0.0)) throw OtError{OTPRG_PARAMETER, "sinkhorn: reg must be positive"};
  if (!(cfg->tol > 0.0)) throw OtError{OTPRG_PARAMETER, "sinkhorn: tol must be positive"};
  OT_CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  const int n_a = p->n_a, n_b = p->n_b;
  const size_t nn = static_cast<size_t>(n_a) * n_b;
  cudaStream_t s = ctx->stream;
  Timer t_build;
  OT_CK(ctx->stage.ensure(nn * 8), "alloc cost");
  OT_CK(ctx->sk_K.ensure(nn * 8), "alloc kernel");
  OT_CK(ctx->sk_P.ensure(nn * 8), "alloc plan");
  // vectors: u, u_next, v, mu, nu, term, row, col, rs, cs, ones, rcost (12 x max n)
  const size_t nm = static_cast<size_t>(std::max(n_a, n_b));
  OT_CK(ctx->sk_vec.ensure(12 * nm * 8 + 64), "alloc vectors");
  OT_CK(ctx->sk_part.ensure(otprg::sk_partial_elems(n_a, n_b) * 8), "alloc partials");
  OT_CK(ctx->sk_int.ensure((nm * 3 + 16) * 8), "alloc flags");
  double* V = ctx->sk_vec.as<double>();
  double *u = V, *u_next = V + nm, *v = V + 2 * nm, *mu = V + 3 * nm, *nu = V + 4 * nm,
         *term = V + 5 * nm, *row = V + 6 * nm, *col = V + 7 * nm, *rs = V + 8 * nm, *cs = V + 9 * nm,
         *ones = V + 10 * nm, *rcost = V + 11 * nm, *scalar = V + 12 * nm;
  int* I = ctx->sk_int.as<int>();
  int *row_ok = I, *col_ok = I + nm, *err = I + 2 * nm, *bad = I + 2 * nm + 4;
  long long* rcnt = reinterpret_cast<long long*>(I + 2 * nm + 16);
  double* cost = ctx->stage.as<double>();
  double* K = ctx->sk_K.as<double>();
  double* P = ctx->sk_P.as<double>();
  OT_CK(otprg::h2d_large(ctx, cost, p->cost, nn * 8), "H2D cost");
  OT_CK(cudaMemcpyAsync(mu, p->mu, n_a * 8ull, cudaMemcpyHostToDevice, s), "H2D mu");
  OT_CK(cudaMemcpyAsync(nu, p->nu, n_b * 8ull, cudaMemcpyHostToDevice, s), "H2D nu");
  OT_CK(cudaMemsetAsync(err, 0, 32, s), "memset");
  OT_CK(otprg::sk_build(cost, n_a, n_b, cfg->reg, K, row_ok, col_ok, bad, s), "kernel build");
  {
    std::vector<int> rok(n_a), cok(n_b);
    int hbad = 0;
    OT_CK(cudaMemcpyAsync(rok.data(), row_ok, n_a * 4ull, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(cok.data(), col_ok, n_b * 4ull, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaStreamSynchronize(s), "kernel build");
    if (hbad) throw OtError{OTPRG_PARAMETER, "OT cost entry outside [0,1]"};
    for (int a = 0; a < n_a; ++a)
      if (!rok[a]) throw OtError{OTPRG_NUMERICAL, "regularization too small: kernel row underflowed"};
    for (int b = 0; b < n_b; ++b)
      if (!cok[b]) throw OtError{OTPRG_NUMERICAL, "regularization too small: kernel column underflowed"};
  }
  r->build_ms = t_build.ms();
  Timer t_loop;
  // u = v = 1 (sinkhorn.cpp:97); the first u-update reads K v0
  std::vector<double> one(nm, 1.0);
  OT_CK(cudaMemcpyAsync(u, one.data(), n_a * 8ull, cudaMemcpyHostToDevice, s), "H2D");
  OT_CK(cudaMemcpyAsync(v, one.data(), n_b * 8ull, cudaMemcpyHostToDevice, s), "H2D");
  OT_CK(otprg::sk_row(K, n_a, n_b, u, v, mu, nullptr, u_next, err, s), "row pass");
  int iters = 0;
  bool converged = false;
  double violation = 0.0;
  auto raise_err = [](int e) {
    if (e & 1) throw OtError{OTPRG_NUMERICAL, "regularization too small: scaling underflowed"};
    if (e & 2) throw OtError{OTPRG_NUMERICAL, "regularization too small: scaling diverged"};
    if (e & 4) throw OtError{OTPRG_NUMERICAL, "regularization too small: scaling underflowed"};
    if (e & 8) throw OtError{OTPRG_NUMERICAL, "regularization too small: scaling diverged"};
  };
  // pinned per-iteration readback: [0] u-update bits, [1] v-update bits, [2..3] violation
  if (ctx->ot_hpin_n < 64) {
    if (ctx->ot_hpin) cudaFreeHost(ctx->ot_hpin);
    ctx->ot_hpin = nullptr;
    ctx->ot_hpin_n = 0;
    OT_CK(cudaMallocHost(&ctx->ot_hpin, 64), "pinned staging");
    ctx->ot_hpin_n = 64;
  }
  int* hb = static_cast<int*>(ctx->ot_hpin);
  while (iters < cfg->max_iters) {
    iters += 1;
    std::swap(u, u_next);  // u-update (computed by the previous row pass; its bits in err[0])
    OT_CK(cudaMemcpyAsync(err + 2, err, 4, cudaMemcpyDeviceToDevice, s), "save bits");
    OT_CK(cudaMemsetAsync(err, 0, 8, s), "memset");
    OT_CK(otprg::sk_col(K, n_a, n_b, u, nu, v, ctx->sk_part.as<double>(), err + 1, s), "col pass");
    // violation of (u, v) and the next u-update from the same K v (bits -> err[0])
    OT_CK(otprg::sk_row(K, n_a, n_b, u, v, mu, term, u_next, err, s), "row pass");
    OT_CK(otprg::sk_sum(term, n_a, scalar, s), "violation");
    OT_CK(cudaMemcpyAsync(hb, err + 1, 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(hb + 2, scalar, 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaStreamSynchronize(s), "sinkhorn iteration");
    raise_err(hb[1] & 3);   // this iteration's u-update (sinkhorn.cpp:110-118)
    raise_err(hb[0] & 12);  // its v-update (:120-128)
    double viol;
    std::memcpy(&viol, hb + 2, 8);
    violation = viol;
    if (violation <= cfg->tol) {
      converged = true;
      break;
    }
    if (cfg->time_budget_ms > 0.0 && t_loop.ms() > cfg->time_budget_ms) break;
  }
  r->iters = iters;
  r->converged = converged ? 1 : 0;
  r->marginal_violation = violation;
  r->loop_ms = t_loop.ms();

  // round_to_marginals (sinkhorn.cpp:12-66) on P = u K v
  Timer t_round;
  OT_CK(otprg::sk_plan(K, n_a, n_b, u, v, nullptr, nullptr, P, s), "plan");
  OT_CK(otprg::sk_prow(P, n_a, n_b, mu, row, rs, s), "row sums");
  OT_CK(otprg::sk_plan(K, n_a, n_b, u, v, rs, nullptr, P, s), "plan");
  OT_CK(otprg::sk_pcol(P, n_a, n_b, ones, ctx->sk_part.as<double>(), col, s), "col sums");
  OT_CK(otprg::sk_colscale(col, nu, n_b, cs, s), "col scale");
  OT_CK(otprg::sk_plan(K, n_a, n_b, u, v, rs, cs, P, s), "plan");
  OT_CK(otprg::sk_prow(P, n_a, n_b, mu, row, nullptr, s), "row sums");
  OT_CK(otprg::sk_pcol(P, n_a, n_b, ones, ctx->sk_part.as<double>(), col, s), "col sums");
  std::vector<double> hrow(n_a), hcol(n_b);
  OT_CK(cudaMemcpyAsync(hrow.data(), row, n_a * 8ull, cudaMemcpyDeviceToHost, s), "D2H");
  OT_CK(cudaMemcpyAsync(hcol.data(), col, n_b * 8ull, cudaMemcpyDeviceToHost, s), "D2H");
  OT_CK(cudaStreamSynchronize(s), "round");
  // greedy placement of the missing mass by index (:50-62)
  std::vector<double> err_a(n_a);
  for (int a = 0; a < n_a; ++a) err_a[a] = std::max(0.0, p->mu[a] - hrow[a]);
  std::vector<int2> add_ab;
  std::vector<double> add_v;
  int a0 = 0;
  for (int b = 0; b < n_b; ++b) {
    double rest = std::max(0.0, p->nu[b] - hcol[b]);
    while (a0 < n_a && !(err_a[a0] > 0.0)) ++a0;
    for (int a = a0; a < n_a && rest > 0.0; ++a) {
      const double add = std::min(err_a[a], rest);
      if (add <= 0.0) continue;
      add_ab.push_back(make_int2(a, b));
      add_v.push_back(add);
      err_a[a] -= add;
      rest -= add;
    }
  }
  if (!add_ab.empty()) {
    OT_CK(ctx->v_k.ensure(add_ab.size() * (sizeof(int2) + 8)), "alloc adds");
    int2* d_ab = reinterpret_cast<int2*>(ctx->v_k.p);
    double* d_add = reinterpret_cast<double*>(d_ab + add_ab.size());
    OT_CK(cudaMemcpyAsync(d_ab, add_ab.data(), add_ab.size() * sizeof(int2), cudaMemcpyHostToDevice, s),
          "H2D");
    OT_CK(cudaMemcpyAsync(d_add, add_v.data(), add_v.size() * 8, cudaMemcpyHostToDevice, s), "H2D");
    OT_CK(otprg::sk_adds(P, n_b, d_ab, d_add, static_cast<int>(add_ab.size()), s), "adds");
  }
  // entries p > 0 (row-major) and the plan cost (:64-72)
  OT_CK(otprg::sk_rowcost(P, cost, n_a, n_b, rcost, rcnt, s), "row cost");
  std::vector<double> hrc(n_a);
  std::vector<long long> hcnt(n_a);
  OT_CK(cudaMemcpyAsync(hrc.data(), rcost, n_a * 8ull, cudaMemcpyDeviceToHost, s), "D2H");
  OT_CK(cudaMemcpyAsync(hcnt.data(), rcnt, n_a * 8ull, cudaMemcpyDeviceToHost, s), "D2H");
  OT_CK(cudaStreamSynchronize(s), "plan cost");
  double total = 0.0;
  std::vector<long long> offs(static_cast<size_t>(n_a) + 1, 0);
  for (int a = 0; a < n_a; ++a) {
    total += hrc[a];
    offs[a + 1] = offs[a] + hcnt[a];
  }
  r->cost = total;
  r->n_entries = offs[n_a];
  if (r->ent_a && r->entry_cap >= r->n_entries && r->n_entries > 0) {
    const size_t ne = static_cast<size_t>(r->n_entries);
    OT_CK(ctx->adm_off.ensure((static_cast<size_t>(n_a) + 1) * 8), "alloc");
    OT_CK(ctx->ot_out.ensure(ne * 16), "alloc entries");
    int32_t* ea = ctx->ot_out.as<int32_t>();
    int32_t* eb = ea + ne;
    double* em = reinterpret_cast<double*>(eb + ne);
    OT_CK(cudaMemcpyAsync(ctx->adm_off.p, offs.data(), (n_a + 1) * 8ull, cudaMemcpyHostToDevice, s), "H2D");
    OT_CK(otprg::sk_entries(P, n_a, n_b, ctx->adm_off.as<long long>(), ea, eb, em, s), "entries");
    OT_CK(cudaMemcpyAsync(r->ent_a, ea, ne * 4, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(r->ent_b, eb, ne * 4, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaMemcpyAsync(r->ent_mass, em, ne * 8, cudaMemcpyDeviceToHost, s), "D2H");
    OT_CK(cudaStreamSynchronize(s), "entries");
  }
  r->round_ms = t_round.ms();
}

}  // namespace

namespace {
template <typename F>
int guarded(otprg_ctx* ctx, F&& f) {
  try {
    f();
    return OTPRG_OK;
  } catch (const OtError& e) {
    ctx->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return OTPRG_DEVICE;
  }
}
}  // namespace

extern "C" {

int otprg_ot_scale_and_round(int32_t n_a, int32_t n_b, const double* mu, const double* nu,
                             double eps, int64_t* d, int64_t* s, double* theta) {
  otprg_ot_problem p{};
  p.n_a = n_a;
  p.n_b = n_b;
  p.mu = mu;
  p.nu = nu;
  p.cost = mu;  // masses only: the cost is not inspected here
  try {
    validate_ot(&p);
    const ScaledMasses sm = scale_and_round(&p, eps);
    std::memcpy(d, sm.d.data(), sm.d.size() * 8);
    std::memcpy(s, sm.s.data(), sm.s.size() * 8);
    *theta = sm.theta;
    return OTPRG_OK;
  } catch (const OtError& e) {
    return e.code;
  }
}

int otprg_solve_ot(otprg_ctx* ctx, const otprg_ot_problem* prob, otprg_ot_result* res) {
  return otprg_solve_ot_opts(ctx, prob, nullptr, res);
}

int otprg_solve_ot_opts(otprg_ctx* ctx, const otprg_ot_problem* prob, const otprg_ot_options* opt,
                        otprg_ot_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!res || (!res->ent_a && res->entry_cap > 0)) {
    ctx->err = "result buffers are null";
    return OTPRG_PARAMETER;
  }
  return guarded(ctx, [&] { OtSolver(ctx, prob, res, opt).run(); });
}

int otprg_solve_copy_matching(otprg_ctx* ctx, const otprg_copy_instance* inst, double eps,
                              const otprg_ot_options* opt, otprg_copy_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!res) {
    ctx->err = "result is null";
    return OTPRG_PARAMETER;
  }
  return guarded(ctx, [&] { OtSolver(ctx, nullptr, nullptr, opt).run_copy(inst, eps, res); });
}

int otprg_copy_state(otprg_ctx* ctx, otprg_cluster_state* out) {
  if (!ctx || !out) return OTPRG_PARAMETER;
  if (!ctx->ot_state) {
    ctx->err = "no copy/cluster solve on this context yet";
    return OTPRG_PARAMETER;
  }
  *out = static_cast<const FlatState*>(ctx->ot_state.get())->view();
  return OTPRG_OK;
}

int otprg_check_cluster_state(const otprg_cluster_state* state, const otprg_copy_instance* inst,
                              int32_t which, int64_t* count, char* msgs, int32_t msgs_cap) {
  if (!state || !inst || !inst->k || (which != 0 && which != 1) || state->n_a != inst->n_a ||
      state->n_b != inst->n_b)
    return OTPRG_PARAMETER;
  const auto v = which == 0 ? check_invariant(*state, *inst) : check_feasibility(*state, *inst);
  if (count) *count = static_cast<int64_t>(v.size());
  if (msgs && msgs_cap > 0) {
    std::string m;
    for (const auto& x : v) m += (m.empty() ? "" : "\n") + x;
    const size_t n = std::min(m.size(), static_cast<size_t>(msgs_cap - 1));
    std::memcpy(msgs, m.data(), n);
    msgs[n] = 0;
  }
  return OTPRG_OK;
}

int otprg_plan_from_flow(const otprg_ot_problem* prob, const int64_t* flow, double theta,
                         const int64_t* d, const int64_t* s, otprg_ot_result* res) {
  (void)d;
  (void)s;  // ScaledMasses' counts: plan_from_flow reads theta only (ot.cpp:639-703)
  if (!prob || !flow || !res || !(theta > 0.0) || (!res->ent_a && res->entry_cap > 0)) return OTPRG_PARAMETER;
  try {
    OtSolver(nullptr, prob, res).run_plan(flow, theta);
    return OTPRG_OK;
  } catch (const OtError& e) {
    return e.code;
  }
}

int otprg_sinkhorn(otprg_ctx* ctx, const otprg_ot_problem* prob, const otprg_sinkhorn_config* cfg,
                   otprg_sinkhorn_result* res) {
  if (!ctx) return OTPRG_PARAMETER;
  if (!res || (!res->ent_a && res->entry_cap > 0)) {
    ctx->err = "result buffers are null";
    return OTPRG_PARAMETER;
  }
  try {
    run_sinkhorn(ctx, prob, cfg, res);
    return OTPRG_OK;
  } catch (const OtError& e) {
    ctx->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return OTPRG_DEVICE;
  }
}

int otprg_random_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed, double* mu, double* nu,
                             double* cost) {
  if (n_a < 1 || n_b < 1 || !mu || !nu || !cost) return OTPRG_PARAMETER;
  auto splitmix64 = [](uint64_t x) {  // instances.cpp:41-46
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
  };
  std::mt19937_64 rma(splitmix64(seed ^ 0x8BB84B93962EACC9ULL));
  std::mt19937_64 rmb(splitmix64(seed ^ 0x2545F4914F6CDD1DULL));
  std::mt19937_64 rc(splitmix64(seed));
  auto bounded = [](std::mt19937_64& r, uint64_t m) {  // instances.cpp:25-32
    const uint64_t limit = ~uint64_t{0} - (~uint64_t{0}) % m;
    uint64_t x;
    do {
      x = r();
    } while (x >= limit);
    return x % m;
  };
  // gen_random_ot_rational (instances.cpp:159-191) + OTInstance::renormalize (ot.cpp:91-100)
  std::vector<int64_t> wa(n_a), wb(n_b);
  int64_t ta = 0, tb = 0;
  for (auto& w : wa) ta += (w = static_cast<int64_t>(bounded(rma, 50)) + 1);
  for (auto& w : wb) tb += (w = static_cast<int64_t>(bounded(rmb, 50)) + 1);
  for (int32_t a = 0; a < n_a; ++a) mu[a] = static_cast<double>(wa[a]) / static_cast<double>(ta);
  for (int32_t b = 0; b < n_b; ++b) nu[b] = static_cast<double>(wb[b]) / static_cast<double>(tb);
  for (size_t i = 0; i < static_cast<size_t>(n_a) * n_b; ++i)
    cost[i] = static_cast<double>(rc() >> 11) * 0x1.0p-53;
  double sum_mu = 0.0, sum_nu = 0.0;
  for (int32_t a = 0; a < n_a; ++a) sum_mu += mu[a];
  for (int32_t b = 0; b < n_b; ++b) sum_nu += nu[b];
  for (int32_t a = 0; a < n_a; ++a) mu[a] /= sum_mu;
  for (int32_t b = 0; b < n_b; ++b) nu[b] /= sum_nu;
  return OTPRG_OK;
}

}  // extern "C"
