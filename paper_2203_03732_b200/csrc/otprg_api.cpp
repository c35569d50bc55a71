// otprg_api.cpp — the C++ API of include/otprg.hpp (the reference's otpr API
// restated in namespace otprg) on top of the C ABI of include/otprg.h.
// Host code only; every solve runs on the device through the C ABI.
#include "../../include/otprg.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <set>
#include <string>
#include <tuple>

#include "../../include/otprg.h"

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
  const otprg_problem p = problem_of(inst, opt.eps, opt.storage);
  ResultBufs rb(inst.n_a, inst.n_b, opt.eps);
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
std::pair<TransportPlan, SolveStats> solve_ot(const OTInstance& inst, double eps) {
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
  std::int64_t cap = 4 * (static_cast<std::int64_t>(p.n_a) + p.n_b) + 64;
  std::vector<std::int64_t> fc(1 << 16);
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
    check(otprg_solve_ot(ctx, &p, &r), ctx);
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
