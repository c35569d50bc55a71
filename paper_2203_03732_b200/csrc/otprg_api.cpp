// otprg_api.cpp — the C++ API of include/otprg.hpp (the reference's otpr API
// restated in namespace otprg) on top of the C ABI of include/otprg.h.
// Host code only; every solve runs on the device through the C ABI.
#include "../../include/otprg.hpp"

#include <algorithm>
#include <exception>
#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <tuple>

#include "../../include/otprg.h"

#include <cuda_runtime.h>

namespace otprg {

namespace {

// One context per (host thread, device), created on first use (a context is
// single-owner like the reference solver).
struct CtxHolder {
  std::map<int, otprg_ctx*> by_dev;
  ~CtxHolder() {
    for (auto& kv : by_dev) otprg_destroy(kv.second);
  }
};

otprg_ctx* context(int device) {
  static thread_local CtxHolder h;
  auto it = h.by_dev.find(device);
  if (it != h.by_dev.end()) return it->second;
  otprg_ctx* c = nullptr;
  if (otprg_create(device, &c) != OTPRG_OK)
    throw DeviceError("otprg: cannot create a context on CUDA device " + std::to_string(device));
  h.by_dev[device] = c;
  return c;
}

[[noreturn]] void raise(int st, otprg_ctx* ctx) {
  const std::string msg = ctx ? otprg_last_error(ctx) : "otprg failure";
  switch (st) {
    case OTPRG_PARAMETER: throw ParameterError(msg);
    case OTPRG_INPUT: throw InputError(msg);
    case OTPRG_NUMERICAL: throw NumericalError(msg);
    case OTPRG_INVARIANT: throw InvariantViolation(msg);
    default: throw DeviceError(msg);
  }
}

void check(int st, otprg_ctx* ctx) {
  if (st != OTPRG_OK) raise(st, ctx);
}

otprg_problem problem_of(const AssignmentInstance& inst, double eps, int storage) {
  otprg_problem p{};
  p.n_a = inst.n_a;
  p.n_b = inst.n_b;
  p.eps = eps;
  p.storage = storage;
  if (inst.cost.size() > 0) {
    if (inst.cost.rows() != inst.n_a || inst.cost.cols() != inst.n_b)
      throw ParameterError("cost matrix dimensions do not match n_a x n_b");
    p.cost_kind = OTPRG_COST_DENSE_F64;
    p.cost = inst.cost.data();
  } else if (!inst.pts_a.empty() || !inst.pts_b.empty()) {
    if (inst.pts_a.size() != 2 * static_cast<size_t>(inst.n_a) ||
        inst.pts_b.size() != 2 * static_cast<size_t>(inst.n_b))
      throw ParameterError("point sets do not match n_a / n_b");
    p.cost_kind = OTPRG_COST_POINTS2D;
    p.pts_a = inst.pts_a.data();
    p.pts_b = inst.pts_b.data();
  } else {
    throw ParameterError("cost matrix dimensions do not match n_a x n_b");
  }
  return p;
}

// gen_uniform_square's cost of one pair (instances.cpp:70-75), non-fused.
double point_cost(const AssignmentInstance& inst, Index a, Index b) {
  const double dx = inst.pts_a[2 * a] - inst.pts_b[2 * b];
  const double dy = inst.pts_a[2 * a + 1] - inst.pts_b[2 * b + 1];
  return std::sqrt(dx * dx + dy * dy) / std::sqrt(2.0);
}

// Caller-side buffers of one otprg_result.
struct ResultBufs {
  Matching m;
  std::vector<std::int64_t> ya, yb, fc;
  otprg_result r{};
  ResultBufs(Index n_a, Index n_b, double eps) : m(n_a, n_b) {
    const Index ia = std::max(n_a, n_b), ib = std::min(n_a, n_b);
    ya.assign(ia, 0);
    yb.assign(ib, 0);
    SolveStats s;
    fc.assign(static_cast<size_t>(std::min<std::int64_t>(s.phase_bound(eps) + 10, OTPRG_MAX_PHASES + 2)), 0);
    r.match_of_a = m.match_of_a.data();
    r.match_of_b = m.match_of_b.data();
    r.y_a = ya.data();
    r.y_b = yb.data();
    r.free_counts = fc.data();
    r.free_cap = static_cast<std::int64_t>(fc.size());
  }
  std::pair<Matching, SolveStats> take() {
    SolveStats s;
    s.phases = static_cast<int>(r.phases);
    s.free_counts.assign(fc.begin(), fc.begin() + std::min<std::int64_t>(r.phases, fc.size()));
    s.sum_ni = r.sum_ni;
    s.duals_final.y_a = ya;
    s.duals_final.y_b = yb;
    s.swapped = r.swapped != 0;
    s.full_match_termination = r.full_match_termination != 0;
    return {m, std::move(s)};
  }
};

const char* kViolation[] = {
    "", "matching is not mutually consistent at a=", "matching is not mutually consistent at b=",
    "demand dual positive at a=", "free demand vertex with nonzero dual at a=",
    "demand dual magnitude exceeds bound at a=", "supply dual negative at b=",
    "supply dual magnitude exceeds bound at b=", "matching edge not tight at (",
    "dual sum exceeds rounded cost allowance at ("};

// verify_feasibility's message strings (assignment.cpp:270-311, core.cpp:69-86)
FeasibilityReport report_of(const otprg_feasibility& f) {
  FeasibilityReport rep;
  if (f.violations == 0) return rep;
  rep.count = f.violations;
  std::string msg = kViolation[f.kind];
  if (f.kind == OTPRG_VIOL_MATCH_B || f.kind == OTPRG_VIOL_SUPPLY_NEGATIVE ||
      f.kind == OTPRG_VIOL_SUPPLY_BOUND)
    msg += std::to_string(f.b);
  else if (f.kind >= OTPRG_VIOL_NOT_TIGHT)
    msg += std::to_string(f.a) + "," + std::to_string(f.b) + "): Y(a)+Y(b)=" + std::to_string(f.sum) +
           " k=" + std::to_string(f.k);
  else
    msg += std::to_string(f.a);
  rep.violations.push_back(msg);
  return rep;
}

Matching internal(const Matching& m, bool swapped) {
  if (!swapped) return m;
  Matching t;
  t.match_of_a = m.match_of_b;
  t.match_of_b = m.match_of_a;
  return t;
}

// The host-synced form of solve_oriented (assignment.cpp:316-364) for
// check_invariants / the observer: one device phase per step.
std::pair<Matching, SolveStats> solve_debug(otprg_ctx* ctx, const AssignmentInstance& inst,
                                            const AssignmentOptions& opt) {
  const otprg_problem p = problem_of(inst, opt.eps, opt.storage);
  const bool swapped = inst.n_b > inst.n_a;
  const bool grouped = opt.demand_groups != nullptr;  // copy mode (assignment.cpp:81-103, :241-250)
  const Index ia = std::max(inst.n_a, inst.n_b), ib = std::min(inst.n_a, inst.n_b);
  ScaledCosts sc;
  if (opt.observer) {  // ScaledCosts in the internal orientation (this also prepares)
    Matrix<std::int32_t> k(inst.n_a, inst.n_b);
    check(otprg_scale_round_costs(ctx, &p, k.data(), &sc.unit_floor, &sc.unit_ceil), ctx);
    sc.eps = opt.eps;
    sc.k = swapped ? k.transposed() : std::move(k);
  } else if (!grouped) {
    otprg_result r{};
    check(otprg_prepare(ctx, &p, &r), ctx);
  }
  if (grouped)
    check(otprg_groups_begin(ctx, &p, opt.demand_groups->data(), opt.supply_groups->data()), ctx);
  else
    check(otprg_begin(ctx), ctx);
  const double threshold = opt.eps * static_cast<double>(ib);
  auto snapshot = [&]() {
    ResultBufs rb(inst.n_a, inst.n_b, opt.eps);
    check(otprg_snapshot(ctx, &rb.r), ctx);
    auto ms = rb.take();
    return std::make_pair(internal(ms.first, swapped), std::move(ms.second.duals_final));
  };
  auto [cur_m, cur_d] = snapshot();
  int phase = 0;
  std::vector<Index> b_free(ib);
  std::vector<std::int64_t> offs(static_cast<size_t>(ib) + 1);
  std::vector<Index> alist;
  while (true) {
    PhaseWorkset ws;
    if (opt.observer) {
      std::int64_t nf = 0, ne = 0;
      check(otprg_admissible(ctx, b_free.data(), offs.data(), nullptr, 0, &nf, &ne), ctx);
      alist.resize(static_cast<size_t>(std::max<std::int64_t>(ne, 1)));
      if (ne > 0) check(otprg_admissible(ctx, b_free.data(), offs.data(), alist.data(), ne, &nf, &ne), ctx);
      ws.b_free.assign(b_free.begin(), b_free.begin() + nf);
      ws.e_admissible.resize(static_cast<size_t>(nf));
      for (std::int64_t i = 0; i < nf; ++i)
        ws.e_admissible[i].assign(alist.begin() + offs[i], alist.begin() + offs[i + 1]);
      if (grouped) {  // scan_grouped order: group, free before matched, partner's group, id
        const auto& dg = *opt.demand_groups;
        const auto& sg = *opt.supply_groups;
        auto key = [&](Index a) {
          const Index b = cur_m.match_of_a[a];
          return std::make_tuple(dg[a], b != kUnmatched ? 1 : 0, b != kUnmatched ? sg[b] : 0, a);
        };
        for (auto& e : ws.e_admissible)
          std::sort(e.begin(), e.end(), [&](Index x, Index y) { return key(x) < key(y); });
      }
    } else {
      for (Index b = 0; b < ib; ++b)
        if (!cur_m.has_b(b)) ws.b_free.push_back(b);
    }
    if (static_cast<double>(ws.b_free.size()) <= threshold) break;
    const DualUnits before = cur_d.sum_abs();
    std::int64_t done = 0;
    std::int32_t fin = 0;
    if (grouped)
      check(otprg_groups_step(ctx, &done, &fin), ctx);
    else
      check(otprg_step(ctx, phase + 1, &done, &fin), ctx);
    if (done != phase + 1)
      throw InvariantViolation("device loop stopped at phase " + std::to_string(done));
    phase = static_cast<int>(done);
    const Matching prev_m = cur_m;
    std::tie(cur_m, cur_d) = snapshot();
    if (opt.check_invariants) {
      otprg_feasibility f{};
      check(otprg_verify_feasibility(ctx, &f), ctx);
      const FeasibilityReport rep = report_of(f);
      if (!rep.ok()) throw InvariantViolation("phase " + std::to_string(phase) + ": " + rep.violations.front());
    }
    if (opt.observer) {
      for (Index b : ws.b_free) {  // M' in B' order, A'' / M'' (apply_phase :214-225)
        const Index a = cur_m.match_of_b[b];
        if (a == kUnmatched) continue;
        ws.m_prime.emplace_back(a, b);
        if (prev_m.match_of_a[a] != kUnmatched) {
          ws.a_double.push_back(a);
          ws.m_double.emplace_back(a, prev_m.match_of_a[a]);
        }
      }
      std::set<Index> touched;
      for (const auto& e : ws.e_admissible) touched.insert(e.begin(), e.end());
      ws.a_touched.assign(touched.begin(), touched.end());
      const PhaseSnapshot snap{phase, sc, cur_d, cur_m, ws, before, cur_d.sum_abs()};
      opt.observer(snap);
    }
  }
  (void)ia;
  ResultBufs rb(inst.n_a, inst.n_b, opt.eps);
  check(grouped ? otprg_groups_finish(ctx, &rb.r) : otprg_finish(ctx, &rb.r), ctx);
  return rb.take();
}

}  // namespace

// ---- core --------------------------------------------------------------------
void AssignmentInstance::validate() const {  // core.cpp:10-24
  if (n_a < 1 || n_b < 1) throw ParameterError("instance needs at least one vertex per side");
  if (cost.size() == 0 && !pts_a.empty()) {
    if (pts_a.size() != 2 * static_cast<size_t>(n_a) || pts_b.size() != 2 * static_cast<size_t>(n_b))
      throw ParameterError("point sets do not match n_a / n_b");
    return;
  }
  if (cost.rows() != n_a || cost.cols() != n_b)
    throw ParameterError("cost matrix dimensions do not match n_a x n_b");
  for (Index a = 0; a < n_a; ++a)
    for (Index b = 0; b < n_b; ++b) {
      const double c = cost(a, b);
      if (!(c >= 0.0 && c <= 1.0))
        throw ParameterError("cost entry outside [0,1] at (" + std::to_string(a) + "," +
                             std::to_string(b) + "): " + std::to_string(c));
    }
}

std::int64_t scaled_floor(double c, double eps) { return otprg_scaled_floor(c, eps); }

ScaledCosts scale_round_costs(const AssignmentInstance& inst, double eps) {
  inst.validate();
  otprg_ctx* ctx = context(0);
  const otprg_problem p = problem_of(inst, eps, 0);
  ScaledCosts sc;
  sc.eps = eps;
  sc.k = Matrix<std::int32_t>(inst.n_a, inst.n_b);
  check(otprg_scale_round_costs(ctx, &p, sc.k.data(), &sc.unit_floor, &sc.unit_ceil), ctx);
  return sc;
}

DualUnits DualState::sum_abs() const {
  DualUnits s = 0;
  for (DualUnits y : y_a) s += std::llabs(y);
  for (DualUnits y : y_b) s += std::llabs(y);
  return s;
}

Index Matching::size() const {
  Index n = 0;
  for (Index b : match_of_a)
    if (b != kUnmatched) ++n;
  return n;
}

void Matching::validate() const {  // core.cpp:69-86
  const auto n_a = static_cast<Index>(match_of_a.size());
  const auto n_b = static_cast<Index>(match_of_b.size());
  for (Index a = 0; a < n_a; ++a) {
    const Index b = match_of_a[a];
    if (b == kUnmatched) continue;
    if (b < 0 || b >= n_b || match_of_b[b] != a)
      throw InvariantViolation("matching is not mutually consistent at a=" + std::to_string(a));
  }
  for (Index b = 0; b < n_b; ++b) {
    const Index a = match_of_b[b];
    if (a == kUnmatched) continue;
    if (a < 0 || a >= n_a || match_of_a[a] != b)
      throw InvariantViolation("matching is not mutually consistent at b=" + std::to_string(b));
  }
}

double matching_cost(const Matching& m, const AssignmentInstance& inst) {  // core.cpp:95-102
  double total = 0.0;
  const bool dense = inst.cost.size() > 0;
  for (Index a = 0; a < inst.n_a; ++a) {
    const Index b = m.match_of_a[a];
    if (b != kUnmatched) total += dense ? inst.cost(a, b) : point_cost(inst, a, b);
  }
  return total;
}

// ---- assignment --------------------------------------------------------------
std::size_t PhaseWorkset::edge_count() const {
  std::size_t n = 0;
  for (const auto& e : e_admissible) n += e.size();
  return n;
}

std::int64_t SolveStats::phase_bound(double eps) const {
  return static_cast<std::int64_t>(std::ceil((1.0 + 2.0 * eps) / (eps * eps)));
}

std::int64_t SolveStats::sum_ni_bound(double eps, Index n) const {
  return static_cast<std::int64_t>(std::ceil(static_cast<double>(n) * (1.0 + 2.0 * eps) / eps));
}

FeasibilityReport verify_feasibility(const ScaledCosts& sc, const DualState& duals, const Matching& m) {
  otprg_ctx* ctx = context(0);
  const Index n_a = sc.k.rows(), n_b = sc.k.cols();
  if (static_cast<Index>(duals.y_a.size()) != n_a || static_cast<Index>(duals.y_b.size()) != n_b ||
      static_cast<Index>(m.match_of_a.size()) != n_a || static_cast<Index>(m.match_of_b.size()) != n_b)
    throw ParameterError("state sizes do not match the cost matrix");
  otprg_feasibility f{};
  check(otprg_verify_host(ctx, n_a, n_b, sc.k.data(), sc.unit_ceil, duals.y_a.data(), duals.y_b.data(),
                          m.match_of_a.data(), m.match_of_b.data(), &f),
        ctx);
  return report_of(f);
}

namespace {
// costs = auto: the rounded matrix (uint16, or uint32 below uint16's eps
// range; rows padded to 256 entries) against the free device memory.
bool on_the_fly(const AssignmentInstance& inst, const AssignmentOptions& opt) {
  if (opt.costs == 2) return true;
  if (opt.costs == 1) return false;
  const size_t ia = std::max(inst.n_a, inst.n_b), ib = std::min(inst.n_a, inst.n_b);
  const double need_units = std::ceil(1.0 / opt.eps) + 2.0;
  const size_t width = opt.storage == OTPRG_STORAGE_U32 || need_units > 65533.0 ? 4 : (opt.storage == OTPRG_STORAGE_U8 ? 1 : 2);
  const size_t need = ib * ((ia + 511) / 512 * 512) * width;
  size_t free_b = 0, total_b = 0;
  if (cudaSetDevice(opt.device) != cudaSuccess || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess)
    return false;
  return static_cast<double>(need) > 0.9 * static_cast<double>(free_b);
}

// Multi-device contexts, one per device list (and thread), kept for reuse.
otprg_ctx* multi_context(const std::vector<int>& devices, int K) {
  static thread_local std::map<std::vector<int>, std::unique_ptr<otprg_ctx, void (*)(otprg_ctx*)>> cache;
  auto it = cache.find(devices);
  if (it == cache.end()) {
    otprg_ctx* c = nullptr;
    std::vector<int32_t> d(devices.begin(), devices.end());
    if (otprg_create_multi(d.data(), static_cast<int32_t>(d.size()), &c) != OTPRG_OK)
      throw DeviceError("otprg: cannot create a multi-device context");
    it = cache.emplace(devices, std::unique_ptr<otprg_ctx, void (*)(otprg_ctx*)>(c, otprg_destroy)).first;
  }
  check(otprg_set_shard_k(it->second.get(), K), it->second.get());
  return it->second.get();
}

// One shard, no kT (OTPRG_FLAG_ON_THE_FLY): the per-phase protocol of
// paper_2203_03732_b200/sharded.py run_phases with a local "exchange".
void solve_on_the_fly(otprg_ctx* ctx, otprg_problem p, otprg_result* r, int device) {
  p.flags |= OTPRG_FLAG_ON_THE_FLY;
  if (cudaSetDevice(device) != cudaSuccess) throw DeviceError("cudaSetDevice");
  const int32_t K = 16, cap = std::min(p.n_a, p.n_b);
  std::int32_t bounds[2];
  check(otprg_shard_prepare(ctx, &p, 1, 0, K, bounds), ctx);
  int32_t *cand = nullptr, *meta = nullptr;
  if (cudaMalloc(&cand, static_cast<size_t>(cap) * K * 4) != cudaSuccess ||
      cudaMalloc(&meta, static_cast<size_t>(cap) * 2 * 4) != cudaSuccess) {
    cudaFree(cand);
    throw DeviceError("on-the-fly solve: candidate buffers");
  }
  struct Free {
    int32_t *c, *m;
    ~Free() {
      cudaFree(c);
      cudaFree(m);
    }
  } guard{cand, meta};
  check(otprg_shard_begin(ctx), ctx);
  while (true) {
    int32_t n = 0, fin = 0;
    check(otprg_shard_top(ctx, &n, &fin), ctx);
    if (fin) break;
    check(otprg_shard_scan(ctx, cand, meta, n, 0), ctx);
    int32_t parked = 0;
    check(otprg_shard_da(ctx, cand, meta, n, 0, &parked), ctx);
    while (parked > 0) {
      check(otprg_shard_scan(ctx, cand, meta, n, 1), ctx);
      check(otprg_shard_da(ctx, cand, meta, n, 1, &parked), ctx);
    }
  }
  check(otprg_shard_finish(ctx, r), ctx);
}
}  // namespace

std::pair<Matching, SolveStats> solve_assignment(const AssignmentInstance& inst,
                                                 const AssignmentOptions& opt) {
  inst.validate();
  if (!(opt.eps > 0.0 && opt.eps < 1.0)) throw ParameterError("eps must lie in (0, 1)");
  if ((opt.demand_groups == nullptr) != (opt.supply_groups == nullptr))
    throw ParameterError("copy mode needs both demand and supply groups");
  if (opt.demand_groups) {  // assignment.cpp:375-381
    if (static_cast<Index>(opt.demand_groups->size()) != inst.n_a ||
        static_cast<Index>(opt.supply_groups->size()) != inst.n_b)
      throw ParameterError("group map sizes do not match the instance");
    if (inst.n_b > inst.n_a) throw ParameterError("copy mode requires n_b <= n_a");
  }
  otprg_ctx* ctx = context(opt.device);
  if (opt.observer || opt.check_invariants || opt.demand_groups) return solve_debug(ctx, inst, opt);
  otprg_problem p = problem_of(inst, opt.eps, opt.storage);
  ResultBufs rb(inst.n_a, inst.n_b, opt.eps);
  if (!opt.devices.empty() && p.cost_kind == OTPRG_COST_POINTS2D) {  // A rows sharded over the devices
    otprg_ctx* mc = multi_context(opt.devices, opt.shard_k);
    if (opt.costs == 2 || (opt.costs == 0 && on_the_fly(inst, opt))) p.flags |= OTPRG_FLAG_ON_THE_FLY;
    check(otprg_solve_assignment(mc, &p, &rb.r), mc);
    return rb.take();
  }
  if ((p.cost_kind == OTPRG_COST_POINTS2D || p.cost_kind == OTPRG_COST_L1_U8) && on_the_fly(inst, opt)) {
    solve_on_the_fly(ctx, p, &rb.r, opt.device);
    return rb.take();
  }
  check(otprg_solve_assignment(ctx, &p, &rb.r), ctx);
  return rb.take();
}

AssignmentInstance gen_uniform_square(Index n, std::uint64_t seed) {  // instances.cpp:48-78
  if (n < 1) throw ParameterError("gen_uniform_square: n must be >= 1");
  AssignmentInstance inst;
  inst.n_a = inst.n_b = n;
  inst.pts_a.resize(2 * static_cast<size_t>(n));
  inst.pts_b.resize(2 * static_cast<size_t>(n));
  check(otprg_uniform_square_points(n, seed, inst.pts_a.data(), inst.pts_b.data()), nullptr);
  inst.cost = Matrix<double>(n, n);
  for (Index a = 0; a < n; ++a)
    for (Index b = 0; b < n; ++b) inst.cost(a, b) = point_cost(inst, a, b);
  inst.norm_factor = std::sqrt(2.0);
  inst.seed = seed;
  return inst;
}

// ---- OT ---------------------------------------------------------------------------
namespace {

// Flat ClusterState (otprg_cluster_state) <-> the reference-shaped types.
ClusterState state_of(const otprg_cluster_state& st) {
  ClusterState s;
  s.demand.resize(st.n_a);
  s.supply.resize(st.n_b);
  for (Index a = 0; a < st.n_a; ++a)
    for (std::int32_t c = st.dem_off[a]; c < st.dem_off[a + 1]; ++c) {
      DemandCluster d;
      d.y = st.dem_y[c];
      d.free_count = st.dem_free[c];
      for (std::int64_t f = st.flow_off[c]; f < st.flow_off[c + 1]; ++f) d.flow.emplace_back(st.flow_b[f], st.flow_cnt[f]);
      s.demand[a].push_back(std::move(d));
    }
  for (Index b = 0; b < st.n_b; ++b)
    for (std::int32_t c = st.sup_off[b]; c < st.sup_off[b + 1]; ++c)
      s.supply[b].push_back(SupplyCluster{st.sup_y[c], st.sup_free[c], st.sup_matched[c]});
  return s;
}

struct FlatOf {
  std::vector<std::int32_t> dem_off{0}, flow_b, sup_off{0};
  std::vector<std::int64_t> dem_y, dem_free, flow_off{0}, flow_cnt, sup_y, sup_free, sup_matched;
  otprg_cluster_state v{};
  explicit FlatOf(const ClusterState& s) {
    for (const auto& cs : s.demand) {
      for (const auto& c : cs) {
        dem_y.push_back(c.y);
        dem_free.push_back(c.free_count);
        for (const auto& [b, n] : c.flow) flow_b.push_back(b), flow_cnt.push_back(n);
        flow_off.push_back(static_cast<std::int64_t>(flow_b.size()));
      }
      dem_off.push_back(static_cast<std::int32_t>(dem_y.size()));
    }
    for (const auto& cs : s.supply) {
      for (const auto& c : cs) sup_y.push_back(c.y), sup_free.push_back(c.free_count), sup_matched.push_back(c.matched_count);
      sup_off.push_back(static_cast<std::int32_t>(sup_y.size()));
    }
    v = otprg_cluster_state{static_cast<std::int32_t>(s.demand.size()), static_cast<std::int32_t>(s.supply.size()),
                            dem_off.data(), dem_y.data(), dem_free.data(), flow_off.data(), flow_b.data(),
                            flow_cnt.data(), sup_off.data(), sup_y.data(), sup_free.data(), sup_matched.data()};
  }
};

otprg_copy_instance flat_instance(const CopyInstance& ci) {
  return otprg_copy_instance{ci.costs.k.rows(), ci.costs.k.cols(), ci.costs.k.data(), ci.costs.unit_ceil,
                             ci.demand_copies.data(), ci.supply_copies.data()};
}

CopyInstance instance_of(const otprg_copy_instance& in) {
  CopyInstance ci;
  ci.costs.k = Matrix<std::int32_t>(in.n_a, in.n_b);
  std::copy(in.k, in.k + static_cast<size_t>(in.n_a) * in.n_b, ci.costs.k.data());
  ci.costs.unit_floor = ci.costs.unit_ceil = static_cast<std::int32_t>(in.unit_ceil);
  ci.demand_copies.assign(in.demand_copies, in.demand_copies + in.n_a);
  ci.supply_copies.assign(in.supply_copies, in.supply_copies + in.n_b);
  return ci;
}

// The observer trampoline: C callback -> std::function, exceptions parked and
// rethrown once the C call has returned (OTPRG_ABORTED).
struct Hooks {
  std::function<void(const ClusterPhaseSnapshot&)> fn;
  const CopyInstance* inst = nullptr;  // the caller's (solve_copy_matching) or built once
  CopyInstance built;
  std::exception_ptr err;
  static int call(const otprg_cluster_snapshot* sn, void* user) {
    Hooks* h = static_cast<Hooks*>(user);
    try {
      if (!h->inst) {
        h->built = instance_of(sn->inst);
        h->inst = &h->built;
      }
      const ClusterState st = state_of(sn->state);
      const ClusterPhaseSnapshot snap{static_cast<int>(sn->phase), *h->inst, st, sn->n_i, sn->sum_abs_before,
                                      sn->sum_abs_after};
      h->fn(snap);
      return 0;
    } catch (...) {
      h->err = std::current_exception();
      return 1;
    }
  }
};

void check_hooks(int st, otprg_ctx* ctx, const Hooks& h) {
  if (st == OTPRG_ABORTED && h.err) std::rethrow_exception(h.err);
  check(st, ctx);
}

std::int64_t free_cap_for(double eps) {
  if (!(eps > 0.0 && eps < 1.0)) return 16;
  SolveStats s;
  return std::min<std::int64_t>(s.phase_bound(eps) + 16, OTPRG_MAX_PHASES + 2);
}

}  // namespace

std::int64_t ScaledMasses::total_d() const {
  std::int64_t t = 0;
  for (auto v : d) t += v;
  return t;
}
std::int64_t ScaledMasses::total_s() const {
  std::int64_t t = 0;
  for (auto v : s) t += v;
  return t;
}
std::int64_t CopyInstance::total_demand() const {
  std::int64_t t = 0;
  for (auto v : demand_copies) t += v;
  return t;
}
std::int64_t CopyInstance::total_supply() const {
  std::int64_t t = 0;
  for (auto v : supply_copies) t += v;
  return t;
}
std::int64_t DemandCluster::matched() const {
  std::int64_t t = 0;
  for (const auto& e : flow) t += e.second;
  return t;
}
Matrix<std::int64_t> ClusterState::flow_matrix(Index n_a, Index n_b) const {
  Matrix<std::int64_t> f(n_a, n_b, 0);
  for (Index a = 0; a < n_a; ++a)
    for (const DemandCluster& c : demand[a])
      for (const auto& [b, cnt] : c.flow) f(a, b) += cnt;
  return f;
}
std::int64_t ClusterState::free_supply_total() const {
  std::int64_t t = 0;
  for (const auto& cs : supply)
    for (const auto& c : cs) t += c.free_count;
  return t;
}
std::int64_t ClusterState::free_demand_of(Index a) const {
  std::int64_t t = 0;
  for (const auto& c : demand[a]) t += c.free_count;
  return t;
}
DualUnits ClusterState::sum_abs_duals() const {
  DualUnits t = 0;
  for (const auto& cs : demand)
    for (const auto& c : cs) t += std::llabs(c.y) * c.count();
  for (const auto& cs : supply)
    for (const auto& c : cs) t += std::llabs(c.y) * c.count();
  return t;
}

ScaledMasses scale_and_round(const OTInstance& inst, double eps) {
  ScaledMasses sm;
  sm.d.resize(inst.n_a());
  sm.s.resize(inst.n_b());
  const int st = otprg_ot_scale_and_round(inst.n_a(), inst.n_b(), inst.mu.data(), inst.nu.data(), eps,
                                          sm.d.data(), sm.s.data(), &sm.theta);
  if (st == OTPRG_PARAMETER) throw ParameterError("scale_and_round: bad masses or eps");
  if (st == OTPRG_INPUT) throw InputError("scale_and_round: masses do not sum to one");
  if (st) throw InvariantViolation("scale_and_round failed");
  return sm;
}

static ClusterReport check_flat(const ClusterState& state, const CopyInstance& inst, int which) {
  const FlatOf f(state);
  const otprg_copy_instance in = flat_instance(inst);
  std::int64_t n = 0;
  std::vector<char> buf(1 << 16);
  if (otprg_check_cluster_state(&f.v, &in, which, &n, buf.data(), static_cast<std::int32_t>(buf.size())) != OTPRG_OK)
    throw ParameterError("cluster state does not match the copy instance");
  ClusterReport r;
  std::string all(buf.data());
  size_t pos = 0;
  for (std::int64_t i = 0; i < n; ++i) {
    const size_t e = all.find('\n', pos);
    r.violations.push_back(all.substr(pos, e == std::string::npos ? std::string::npos : e - pos));
    if (e == std::string::npos) break;
    pos = e + 1;
  }
  while (static_cast<std::int64_t>(r.violations.size()) < n) r.violations.emplace_back("(truncated)");
  return r;
}
ClusterReport check_cluster_invariant(const ClusterState& state, const CopyInstance& inst) {
  return check_flat(state, inst, 0);
}
ClusterReport check_cluster_feasibility(const ClusterState& state, const CopyInstance& inst) {
  return check_flat(state, inst, 1);
}

ClusterSolveResult solve_copy_matching(const CopyInstance& inst, double eps, const ClusterOptions& opt) {
  otprg_ctx* ctx = context(0);
  const otprg_copy_instance in = flat_instance(inst);
  if (inst.costs.k.rows() != static_cast<Index>(inst.demand_copies.size()) ||
      inst.costs.k.cols() != static_cast<Index>(inst.supply_copies.size()))
    throw ParameterError("copy counts do not match the cost matrix");
  Hooks h;
  h.fn = opt.observer;
  h.inst = &inst;
  otprg_ot_options o{opt.check_invariants ? 1 : 0, 0, opt.observer ? &Hooks::call : nullptr, &h};
  ClusterSolveResult res;
  res.flow = Matrix<std::int64_t>(in.n_a, in.n_b, 0);
  std::vector<std::int64_t> fc(static_cast<size_t>(free_cap_for(eps)));
  otprg_copy_result r{};
  r.flow = res.flow.data();
  r.free_counts = fc.data();
  r.free_cap = static_cast<std::int64_t>(fc.size());
  check_hooks(otprg_solve_copy_matching(ctx, &in, eps, &o, &r), ctx, h);
  otprg_cluster_state st{};
  check(otprg_copy_state(ctx, &st), ctx);
  res.state = state_of(st);
  res.stats.phases = static_cast<int>(r.phases);
  res.stats.free_counts.assign(fc.begin(), fc.begin() + std::min<std::int64_t>(r.phases, fc.size()));
  res.stats.sum_ni = r.sum_ni;
  res.stats.full_match_termination = r.full_match_termination != 0;
  return res;
}

TransportPlan plan_from_flow(const Matrix<std::int64_t>& flow, const ScaledMasses& sm, const OTInstance& inst) {
  if (flow.rows() != inst.n_a() || flow.cols() != inst.n_b())
    throw ParameterError("flow matrix dimensions do not match the instance");
  otprg_ot_problem p{};
  p.n_a = inst.n_a();
  p.n_b = inst.n_b();
  p.eps = 0.5;
  p.mu = inst.mu.data();
  p.nu = inst.nu.data();
  p.cost = inst.cost.data();
  std::int64_t cap = static_cast<std::int64_t>(flow.size()) + p.n_a + p.n_b + 16;
  std::vector<std::int32_t> ea(cap), eb(cap);
  std::vector<double> em(cap);
  otprg_ot_result r{};
  r.ent_a = ea.data();
  r.ent_b = eb.data();
  r.ent_mass = em.data();
  r.entry_cap = cap;
  const int st = otprg_plan_from_flow(&p, flow.data(), sm.theta, sm.d.data(), sm.s.data(), &r);
  if (st == OTPRG_PARAMETER) throw ParameterError("plan_from_flow: bad flow or instance");
  if (st) throw InvariantViolation("plan_from_flow: residual supply could not be placed");
  TransportPlan plan;
  plan.cost = r.cost;
  plan.entries.resize(static_cast<size_t>(r.n_entries));
  for (std::int64_t i = 0; i < r.n_entries; ++i) plan.entries[i] = {ea[i], eb[i], em[i]};
  return plan;
}

std::pair<TransportPlan, SolveStats> solve_ot(const OTInstance& inst, double eps, const OTOptions& opt) {
  if (inst.cost.rows() != inst.n_a() || inst.cost.cols() != inst.n_b())
    throw ParameterError("OT cost matrix dimensions do not match mass vectors");
  otprg_ctx* ctx = context(0);
  otprg_ot_problem p{};
  p.n_a = inst.n_a();
  p.n_b = inst.n_b();
  p.eps = eps;
  p.mu = inst.mu.data();
  p.nu = inst.nu.data();
  p.cost = inst.cost.data();
  Hooks h;
  h.fn = opt.observer;
  const bool hooks = opt.check_invariants || opt.observer;
  otprg_ot_options o{opt.check_invariants ? 1 : 0, 0, opt.observer ? &Hooks::call : nullptr, &h};
  std::int64_t cap = 4 * (static_cast<std::int64_t>(p.n_a) + p.n_b) + 64;
  if (hooks) cap = std::max<std::int64_t>(cap, static_cast<std::int64_t>(p.n_a) * p.n_b);  // hooks run once
  std::vector<std::int64_t> fc(static_cast<size_t>(free_cap_for(eps / 3.0)));
  for (int attempt = 0; attempt < 2; ++attempt) {
    std::vector<std::int32_t> ea(cap), eb(cap);
    std::vector<double> em(cap);
    otprg_ot_result r{};
    r.ent_a = ea.data();
    r.ent_b = eb.data();
    r.ent_mass = em.data();
    r.entry_cap = cap;
    r.free_counts = fc.data();
    r.free_cap = static_cast<std::int64_t>(fc.size());
    check_hooks(otprg_solve_ot_opts(ctx, &p, hooks && attempt == 0 ? &o : nullptr, &r), ctx, h);
    if (r.n_entries > cap) {  // room for every entry, then once more
      cap = r.n_entries;
      continue;
    }
    TransportPlan plan;
    plan.cost = r.cost;
    plan.entries.resize(static_cast<size_t>(r.n_entries));
    for (std::int64_t i = 0; i < r.n_entries; ++i) plan.entries[i] = {ea[i], eb[i], em[i]};
    SolveStats s;
    s.phases = static_cast<int>(r.phases);
    s.free_counts.assign(fc.begin(), fc.begin() + std::min<std::int64_t>(r.phases, fc.size()));
    s.sum_ni = r.sum_ni;
    s.full_match_termination = r.full_match_termination != 0;
    return {std::move(plan), std::move(s)};
  }
  throw DeviceError("solve_ot: plan size changed between runs");
}

OTInstance gen_random_ot_rational(Index n_a, Index n_b, std::uint64_t seed) {
  OTInstance ot;
  ot.mu.resize(n_a);
  ot.nu.resize(n_b);
  ot.cost = Matrix<double>(n_a, n_b);
  if (otprg_random_ot_rational(n_a, n_b, seed, ot.mu.data(), ot.nu.data(), ot.cost.data()) != OTPRG_OK)
    throw ParameterError("gen_random_ot_rational: sides must be >= 1");
  ot.seed = seed;
  return ot;
}

SinkhornResult sinkhorn(const OTInstance& inst, const SinkhornConfig& cfg) {
  if (inst.cost.rows() != inst.n_a() || inst.cost.cols() != inst.n_b())
    throw ParameterError("OT cost matrix dimensions do not match mass vectors");
  otprg_ctx* ctx = context(0);
  otprg_ot_problem p{};
  p.n_a = inst.n_a();
  p.n_b = inst.n_b();
  p.eps = 0.5;
  p.mu = inst.mu.data();
  p.nu = inst.nu.data();
  p.cost = inst.cost.data();
  otprg_sinkhorn_config c{cfg.reg, cfg.max_iters, 0, cfg.tol, cfg.time_budget_ms};
  otprg_sinkhorn_result r{};
  check(otprg_sinkhorn(ctx, &p, &c, &r), ctx);
  const std::int64_t ne = r.n_entries;
  std::vector<std::int32_t> ea(ne > 0 ? ne : 1), eb(ne > 0 ? ne : 1);
  std::vector<double> em(ne > 0 ? ne : 1);
  otprg_sinkhorn_result r2{};
  r2.ent_a = ea.data();
  r2.ent_b = eb.data();
  r2.ent_mass = em.data();
  r2.entry_cap = ne;
  check(otprg_sinkhorn(ctx, &p, &c, &r2), ctx);
  SinkhornResult out;
  out.plan.cost = r2.cost;
  out.plan.entries.resize(static_cast<size_t>(r2.n_entries));
  for (std::int64_t i = 0; i < r2.n_entries; ++i) out.plan.entries[i] = {ea[i], eb[i], em[i]};
  out.iters = r2.iters;
  out.cost = r2.cost;
  out.converged = r2.converged != 0;
  out.marginal_violation = r2.marginal_violation;
  return out;
}

}  // namespace otprg
