// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libotpr_ref.so).  It lets the Python tests, the golden-fixture
// generator and bench.py's reference arm call the reference's own public API
// (otpr::solve_assignment, otpr::solve_ot, ...) through ctypes.  This file is
// ours; no reference source is copied into the repo.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "otpr/assignment.hpp"
#include "otpr/bench.hpp"
#include "otpr/core.hpp"
#include "otpr/errors.hpp"
#include "otpr/instances.hpp"
#include "otpr/oracles.hpp"
#include "otpr/ot.hpp"
#include "otpr/sinkhorn.hpp"

namespace {

thread_local std::string g_err;

// Exception -> status mapping of tools/otbench.cpp:187-209.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const otpr::ParameterError& e) {
    g_err = e.what();
    return 2;
  } catch (const otpr::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const otpr::InputError& e) {
    g_err = e.what();
    return 3;
  } catch (const otpr::NumericalError& e) {
    g_err = e.what();
    return 4;
  } catch (const otpr::InvariantViolation& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct RefStats {
  int64_t phases;
  int64_t sum_ni;
  int32_t swapped;
  int32_t full_match_termination;
  double cost;
  double solve_ms;  // steady_clock around solve_assignment (bench.cpp:62-64)
  double round_ms;  // scale_round_costs alone, timed separately (untimed solve)
  int64_t n_free_counts;
};

void export_result(const otpr::Matching& m, const otpr::SolveStats& s,
                   int32_t* match_of_a, int32_t* match_of_b, int64_t* y_a,
                   int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                   RefStats* out) {
  if (match_of_a)
    std::memcpy(match_of_a, m.match_of_a.data(), m.match_of_a.size() * 4);
  if (match_of_b)
    std::memcpy(match_of_b, m.match_of_b.data(), m.match_of_b.size() * 4);
  if (y_a)
    std::memcpy(y_a, s.duals_final.y_a.data(), s.duals_final.y_a.size() * 8);
  if (y_b)
    std::memcpy(y_b, s.duals_final.y_b.data(), s.duals_final.y_b.size() * 8);
  const int64_t nf = static_cast<int64_t>(s.free_counts.size());
  if (free_counts)
    std::memcpy(free_counts, s.free_counts.data(),
                static_cast<size_t>(nf < free_cap ? nf : free_cap) * 8);
  out->phases = s.phases;
  out->sum_ni = s.sum_ni;
  out->swapped = s.swapped;
  out->full_match_termination = s.full_match_termination;
  out->n_free_counts = nf;
}

otpr::AssignmentInstance wrap(int32_t n_a, int32_t n_b, const double* cost) {
  otpr::AssignmentInstance inst;
  inst.n_a = n_a;
  inst.n_b = n_b;
  inst.cost = otpr::Matrix<double>(n_a, n_b);
  std::memcpy(inst.cost.data(), cost, sizeof(double) * size_t(n_a) * n_b);
  return inst;
}

int solve_inst(const otpr::AssignmentInstance& inst, double eps, int threads,
               int time_rounding, int32_t* match_of_a, int32_t* match_of_b,
               int64_t* y_a, int64_t* y_b, int64_t* free_counts,
               int64_t free_cap, RefStats* out) {
  return guarded([&] {
    otpr::AssignmentOptions opt;
    opt.eps = eps;
    opt.threads = threads;
    const auto t0 = Clock::now();
    auto [m, s] = otpr::solve_assignment(inst, opt);
    out->solve_ms = ms_since(t0);
    out->cost = otpr::matching_cost(m, inst);
    out->round_ms = 0.0;
    if (time_rounding) {
      const auto t1 = Clock::now();
      volatile auto sc = otpr::scale_round_costs(inst, eps).unit_floor;
      (void)sc;
      out->round_ms = ms_since(t1);
    }
    export_result(m, s, match_of_a, match_of_b, y_a, y_b, free_counts, free_cap,
                  out);
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_gen_uniform_square(int32_t n, uint64_t seed, double* cost) {
  return guarded([&] {
    const auto inst = otpr::gen_uniform_square(n, seed);
    std::memcpy(cost, inst.cost.data(), sizeof(double) * inst.cost.size());
  });
}

int ref_scale_round_costs(int32_t n_a, int32_t n_b, const double* cost,
                          double eps, int32_t* k, int32_t* unit_floor,
                          int32_t* unit_ceil) {
  return guarded([&] {
    const auto sc = otpr::scale_round_costs(wrap(n_a, n_b, cost), eps);
    std::memcpy(k, sc.k.data(), sizeof(int32_t) * sc.k.size());
    *unit_floor = sc.unit_floor;
    *unit_ceil = sc.unit_ceil;
  });
}

int64_t ref_scaled_floor(double c, double eps) { return otpr::scaled_floor(c, eps); }

int ref_solve_assignment(int32_t n_a, int32_t n_b, const double* cost, double eps,
                         int threads, int32_t* match_of_a, int32_t* match_of_b,
                         int64_t* y_a, int64_t* y_b, int64_t* free_counts,
                         int64_t free_cap, RefStats* out) {
  otpr::AssignmentInstance inst;
  int st = guarded([&] { inst = wrap(n_a, n_b, cost); });
  if (st) return st;
  return solve_inst(inst, eps, threads, 0, match_of_a, match_of_b, y_a, y_b,
                    free_counts, free_cap, out);
}

// gen_uniform_square(n, seed) + solve_assignment in one call, so large
// instances never cross the FFI.  gen_ms reports the (untimed-by-reference)
// instance generation.
int ref_solve_uniform_square(int32_t n, uint64_t seed, double eps, int threads,
                             int time_rounding, int32_t* match_of_a,
                             int32_t* match_of_b, int64_t* y_a, int64_t* y_b,
                             int64_t* free_counts, int64_t free_cap,
                             RefStats* out) {
  otpr::AssignmentInstance inst;
  int st = guarded([&] { inst = otpr::gen_uniform_square(n, seed); });
  if (st) return st;
  return solve_inst(inst, eps, threads, time_rounding, match_of_a, match_of_b,
                    y_a, y_b, free_counts, free_cap, out);
}

// load_mnist_pair(path, n, seed): dense cost out (n x n).
int ref_load_mnist_pair(const char* path, int32_t n, uint64_t seed, double* cost) {
  return guarded([&] {
    const auto inst = otpr::load_mnist_pair(path, n, seed);
    std::memcpy(cost, inst.cost.data(), sizeof(double) * inst.cost.size());
  });
}

int ref_solve_mnist(const char* path, int32_t n, uint64_t seed, double eps,
                    int threads, int32_t* match_of_a, int32_t* match_of_b,
                    int64_t* y_a, int64_t* y_b, int64_t* free_counts,
                    int64_t free_cap, RefStats* out, double* load_ms) {
  otpr::AssignmentInstance inst;
  const auto t0 = Clock::now();
  int st = guarded([&] { inst = otpr::load_mnist_pair(path, n, seed); });
  if (load_ms) *load_ms = ms_since(t0);
  if (st) return st;
  return solve_inst(inst, eps, threads, 0, match_of_a, match_of_b, y_a, y_b,
                    free_counts, free_cap, out);
}

// ---- optimal transport (src/ot.cpp:705-732) -------------------------------

struct RefOtStats {
  int64_t phases;
  int64_t sum_ni;
  int64_t n_entries;
  double cost;
  double theta;
  double solve_ms;
  int64_t total_d;
  int64_t total_s;
};

// gen_random_ot_rational(n_a, n_b, seed) -> solve_ot(eps).  Plan entries are
// written up to entry_cap as (a, b, mass) triples.
int ref_solve_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed, double eps,
                          int32_t* ent_a, int32_t* ent_b, double* ent_mass,
                          int64_t entry_cap, int64_t* free_counts,
                          int64_t free_cap, RefOtStats* out) {
  otpr::OTInstance inst;
  int st = guarded([&] { inst = otpr::gen_random_ot_rational(n_a, n_b, seed); });
  if (st) return st;
  return guarded([&] {
    const auto sm = otpr::scale_and_round(inst, eps / 3.0);
    out->theta = sm.theta;
    out->total_d = sm.total_d();
    out->total_s = sm.total_s();
    const auto t0 = Clock::now();
    auto [plan, stats] = otpr::solve_ot(inst, eps);
    out->solve_ms = ms_since(t0);
    out->phases = stats.phases;
    out->sum_ni = stats.sum_ni;
    out->cost = plan.cost;
    out->n_entries = static_cast<int64_t>(plan.entries.size());
    const int64_t ne = out->n_entries < entry_cap ? out->n_entries : entry_cap;
    for (int64_t i = 0; i < ne; ++i) {
      ent_a[i] = plan.entries[i].a;
      ent_b[i] = plan.entries[i].b;
      ent_mass[i] = plan.entries[i].mass;
    }
    const int64_t nf = static_cast<int64_t>(stats.free_counts.size());
    if (free_counts)
      std::memcpy(free_counts, stats.free_counts.data(),
                  static_cast<size_t>(nf < free_cap ? nf : free_cap) * 8);
  });
}

// The OT instance itself (renormalised masses + costs) for parity inputs.
int ref_gen_random_ot_rational(int32_t n_a, int32_t n_b, uint64_t seed,
                               double* mu, double* nu, double* cost) {
  return guarded([&] {
    const auto inst = otpr::gen_random_ot_rational(n_a, n_b, seed);
    std::memcpy(mu, inst.mu.data(), sizeof(double) * inst.mu.size());
    std::memcpy(nu, inst.nu.data(), sizeof(double) * inst.nu.size());
    std::memcpy(cost, inst.cost.data(), sizeof(double) * inst.cost.size());
  });
}

}  // extern "C"

extern "C" {

// solve_ot on a caller-given instance (mu, nu, row-major cost); renormalize()
// is NOT applied (the caller passes masses exactly as the reference would see
// them).
int ref_solve_ot(int32_t n_a, int32_t n_b, const double* mu, const double* nu,
                 const double* cost, double eps, int32_t* ent_a, int32_t* ent_b,
                 double* ent_mass, int64_t entry_cap, int64_t* free_counts,
                 int64_t free_cap, RefOtStats* out) {
  return guarded([&] {
    otpr::OTInstance inst;
    inst.mu.assign(mu, mu + n_a);
    inst.nu.assign(nu, nu + n_b);
    inst.cost = otpr::Matrix<double>(n_a, n_b);
    std::memcpy(inst.cost.data(), cost, sizeof(double) * size_t(n_a) * n_b);
    const auto sm = otpr::scale_and_round(inst, eps / 3.0);
    out->theta = sm.theta;
    out->total_d = sm.total_d();
    out->total_s = sm.total_s();
    const auto t0 = Clock::now();
    auto [plan, stats] = otpr::solve_ot(inst, eps);
    out->solve_ms = ms_since(t0);
    out->phases = stats.phases;
    out->sum_ni = stats.sum_ni;
    out->cost = plan.cost;
    out->n_entries = static_cast<int64_t>(plan.entries.size());
    const int64_t ne = out->n_entries < entry_cap ? out->n_entries : entry_cap;
    for (int64_t i = 0; i < ne; ++i) {
      ent_a[i] = plan.entries[i].a;
      ent_b[i] = plan.entries[i].b;
      ent_mass[i] = plan.entries[i].mass;
    }
    const int64_t nf = static_cast<int64_t>(stats.free_counts.size());
    if (free_counts)
      std::memcpy(free_counts, stats.free_counts.data(),
                  static_cast<size_t>(nf < free_cap ? nf : free_cap) * 8);
  });
}

// scale_and_round(inst, eps): copy counts (ot.cpp:109-128).
int ref_scale_and_round(int32_t n_a, int32_t n_b, const double* mu, const double* nu,
                        const double* cost, double eps, int64_t* d, int64_t* s,
                        double* theta) {
  return guarded([&] {
    otpr::OTInstance inst;
    inst.mu.assign(mu, mu + n_a);
    inst.nu.assign(nu, nu + n_b);
    inst.cost = otpr::Matrix<double>(n_a, n_b);
    std::memcpy(inst.cost.data(), cost, sizeof(double) * size_t(n_a) * n_b);
    const auto sm = otpr::scale_and_round(inst, eps);
    std::memcpy(d, sm.d.data(), 8 * sm.d.size());
    std::memcpy(s, sm.s.data(), 8 * sm.s.size());
    *theta = sm.theta;
  });
}

// format_double (bench.cpp:203-208): the CSV number format.
int ref_format_double(double v, char* out, int32_t cap) {
  const std::string f = otpr::format_double(v);
  if (static_cast<int32_t>(f.size()) + 1 > cap) return 2;
  std::memcpy(out, f.c_str(), f.size() + 1);
  return 0;
}

// csv_row (bench.cpp:214-228) of one record (optional fields: has_* = 0 -> empty).
int ref_csv_row(const char* solver, int32_t n, int32_t has_eps, double eps, int32_t has_reg,
                double reg, uint64_t seed, double cost, int32_t has_oracle, double oracle,
                double time_ms, int64_t phases, char* out, int32_t cap) {
  return guarded([&] {
    otpr::RunRecord r;
    r.solver = solver;
    r.n = n;
    if (has_eps) r.eps = eps;
    if (has_reg) r.reg = reg;
    r.seed = seed;
    r.cost = cost;
    if (has_oracle) r.oracle_cost = oracle;
    r.time_ms = time_ms;
    r.phases = phases;
    const std::string row = otpr::csv_row(r);
    if (static_cast<int32_t>(row.size()) + 1 > cap) throw otpr::ParameterError("buffer");
    std::memcpy(out, row.c_str(), row.size() + 1);
  });
}

// save_instance (instances.cpp:209-222) of gen_uniform_square(n, seed).
int ref_save_uniform_square(int32_t n, uint64_t seed, const char* path) {
  return guarded([&] { otpr::save_instance(otpr::gen_uniform_square(n, seed), path); });
}

// load_instance (instances.cpp:224-246): header + cost.
int ref_load_instance(const char* path, int32_t* n_a, int32_t* n_b, double* norm_factor,
                      uint64_t* seed, double* cost, int64_t cost_cap) {
  return guarded([&] {
    const auto inst = otpr::load_instance(path);
    *n_a = inst.n_a;
    *n_b = inst.n_b;
    *norm_factor = inst.norm_factor;
    *seed = inst.seed;
    if (cost && cost_cap >= static_cast<int64_t>(inst.cost.size()))
      std::memcpy(cost, inst.cost.data(), inst.cost.size() * sizeof(double));
  });
}

// sinkhorn (sinkhorn.cpp:69-151): iters, converged, violation, cost and (when
// cap allows) the plan entries.
int ref_sinkhorn(int32_t n_a, int32_t n_b, const double* mu, const double* nu, const double* cost,
                 double reg, int32_t max_iters, double tol, int32_t* iters, int32_t* converged,
                 double* violation, double* plan_cost, int64_t* n_entries, int32_t* ea, int32_t* eb,
                 double* em, int64_t cap, double* ms) {
  return guarded([&] {
    otpr::OTInstance inst;
    inst.mu.assign(mu, mu + n_a);
    inst.nu.assign(nu, nu + n_b);
    inst.cost = otpr::Matrix<double>(n_a, n_b);
    std::memcpy(inst.cost.data(), cost, sizeof(double) * size_t(n_a) * n_b);
    otpr::SinkhornConfig cfg;
    cfg.reg = reg;
    cfg.max_iters = max_iters;
    cfg.tol = tol;
    const auto t0 = Clock::now();
    const auto res = otpr::sinkhorn(inst, cfg);
    *ms = ms_since(t0);
    *iters = res.iters;
    *converged = res.converged ? 1 : 0;
    *violation = res.marginal_violation;
    *plan_cost = res.cost;
    *n_entries = static_cast<int64_t>(res.plan.entries.size());
    if (ea && cap >= *n_entries)
      for (size_t i = 0; i < res.plan.entries.size(); ++i) {
        ea[i] = res.plan.entries[i].a;
        eb[i] = res.plan.entries[i].b;
        em[i] = res.plan.entries[i].mass;
      }
  });
}

// solve_assignment in copy mode (AssignmentOptions::demand_groups /
// supply_groups, assignment.cpp:81-103, :241-250), threads = 1; with
// check_invariants when asked.
int ref_solve_assignment_groups(int32_t n_a, int32_t n_b, const double* cost, double eps,
                                const int32_t* demand_groups, const int32_t* supply_groups,
                                int32_t check_invariants, int32_t* match_of_a, int32_t* match_of_b,
                                int64_t* y_a, int64_t* y_b, int64_t* free_counts, int64_t free_cap,
                                RefStats* out) {
  return guarded([&] {
    const otpr::AssignmentInstance inst = wrap(n_a, n_b, cost);
    const std::vector<otpr::Index> dg(demand_groups, demand_groups + n_a);
    const std::vector<otpr::Index> sg(supply_groups, supply_groups + n_b);
    otpr::AssignmentOptions opt;
    opt.eps = eps;
    opt.demand_groups = &dg;
    opt.supply_groups = &sg;
    opt.check_invariants = check_invariants != 0;
    const auto t0 = Clock::now();
    auto [m, s] = otpr::solve_assignment(inst, opt);
    out->solve_ms = ms_since(t0);
    out->cost = otpr::matching_cost(m, inst);
    out->round_ms = 0.0;
    export_result(m, s, match_of_a, match_of_b, y_a, y_b, free_counts, free_cap, out);
  });
}

// The reference's exact oracles (oracles.hpp:18-37), used by the acceptance
// checks as the optimum to bound against (test infrastructure only).
int ref_hungarian_exact(int32_t n_a, int32_t n_b, const double* cost, double* opt_cost) {
  return guarded([&] { *opt_cost = otpr::hungarian_exact(wrap(n_a, n_b, cost), 4096).second; });
}

int ref_exact_ot(int32_t n_a, int32_t n_b, const double* mu, const double* nu, const double* cost,
                 double* opt_cost) {
  return guarded([&] {
    otpr::OTInstance inst;
    inst.mu.assign(mu, mu + n_a);
    inst.nu.assign(nu, nu + n_b);
    inst.cost = otpr::Matrix<double>(n_a, n_b);
    std::memcpy(inst.cost.data(), cost, sizeof(double) * size_t(n_a) * n_b);
    *opt_cost = otpr::exact_ot(inst, 256).second;
  });
}


// ---- copy/cluster solver (ot.hpp:52-151), for the OT phase-primitive tests --
static otpr::CopyInstance make_copy(int32_t n_a, int32_t n_b, const int32_t* k, double ceps,
                                    int32_t unit_floor, int32_t unit_ceil, const int64_t* d,
                                    const int64_t* s) {
  otpr::CopyInstance ci;
  ci.costs.eps = ceps;
  ci.costs.unit_floor = unit_floor;
  ci.costs.unit_ceil = unit_ceil;
  ci.costs.k = otpr::Matrix<int32_t>(n_a, n_b);
  std::memcpy(ci.costs.k.data(), k, sizeof(int32_t) * size_t(n_a) * n_b);
  ci.demand_copies.assign(d, d + n_a);
  ci.supply_copies.assign(s, s + n_b);
  return ci;
}

// Flat ClusterState (include/otprg.h otprg_cluster_state layout, counts first):
// sizes[0..2] = clusters (demand), flow entries, clusters (supply).
static void flatten(const otpr::ClusterState& st, int32_t* dem_off, int64_t* dem_y, int64_t* dem_free,
                    int64_t* flow_off, int32_t* flow_b, int64_t* flow_cnt, int32_t* sup_off,
                    int64_t* sup_y, int64_t* sup_free, int64_t* sup_matched, int64_t cap,
                    int64_t* sizes) {
  int64_t nd = 0, nf = 0, ns = 0;
  dem_off[0] = 0;
  flow_off[0] = 0;
  for (size_t a = 0; a < st.demand.size(); ++a) {
    for (const auto& c : st.demand[a]) {
      if (nd < cap) dem_y[nd] = c.y, dem_free[nd] = c.free_count;
      for (const auto& [b, cnt] : c.flow) {
        if (nf < cap) flow_b[nf] = b, flow_cnt[nf] = cnt;
        ++nf;
      }
      ++nd;
      if (nd < cap + 1) flow_off[nd] = nf;
    }
    dem_off[a + 1] = static_cast<int32_t>(nd);
  }
  sup_off[0] = 0;
  for (size_t b = 0; b < st.supply.size(); ++b) {
    for (const auto& c : st.supply[b]) {
      if (ns < cap) sup_y[ns] = c.y, sup_free[ns] = c.free_count, sup_matched[ns] = c.matched_count;
      ++ns;
    }
    sup_off[b + 1] = static_cast<int32_t>(ns);
  }
  sizes[0] = nd, sizes[1] = nf, sizes[2] = ns;
}

// otpr::solve_copy_matching: final flow (completion included), free_counts,
// phases / sum_ni / full_match_termination in stats6[0..2], the per-phase flow
// matrices (observer, up to phase_cap of them) and the final state, flat.
int ref_solve_copy_matching(int32_t n_a, int32_t n_b, const int32_t* k, double ceps,
                            int32_t unit_floor, int32_t unit_ceil, const int64_t* d,
                            const int64_t* s, double eps, int32_t check, int64_t* flow,
                            int64_t* free_counts, int64_t free_cap, int64_t* phase_flows,
                            int64_t phase_cap, int64_t* phase_ni, int64_t* stats3,
                            int32_t* dem_off, int64_t* dem_y, int64_t* dem_free, int64_t* flow_off,
                            int32_t* flow_b, int64_t* flow_cnt, int32_t* sup_off, int64_t* sup_y,
                            int64_t* sup_free, int64_t* sup_matched, int64_t cap, int64_t* sizes) {
  return guarded([&] {
    const otpr::CopyInstance ci = make_copy(n_a, n_b, k, ceps, unit_floor, unit_ceil, d, s);
    otpr::ClusterOptions opt;
    opt.check_invariants = check != 0;
    const size_t nn = size_t(n_a) * n_b;
    opt.observer = [&](const otpr::ClusterPhaseSnapshot& snap) {
      if (snap.phase <= phase_cap) {
        const auto f = snap.state.flow_matrix(n_a, n_b);
        std::memcpy(phase_flows + (snap.phase - 1) * nn, f.data(), nn * 8);
        phase_ni[snap.phase - 1] = snap.n_i;
      }
    };
    const otpr::ClusterSolveResult r = otpr::solve_copy_matching(ci, eps, opt);
    std::memcpy(flow, r.flow.data(), nn * 8);
    const int64_t nf = static_cast<int64_t>(r.stats.free_counts.size());
    std::memcpy(free_counts, r.stats.free_counts.data(), size_t(nf < free_cap ? nf : free_cap) * 8);
    stats3[0] = r.stats.phases;
    stats3[1] = r.stats.sum_ni;
    stats3[2] = r.stats.full_match_termination ? 1 : 0;
    flatten(r.state, dem_off, dem_y, dem_free, flow_off, flow_b, flow_cnt, sup_off, sup_y, sup_free,
            sup_matched, cap, sizes);
  });
}

// otpr::check_cluster_invariant (which 0) / check_cluster_feasibility (1) on a
// flat state: violation count and the messages, newline-separated.
int ref_check_cluster(int32_t n_a, int32_t n_b, const int32_t* k, int32_t unit_ceil,
                      const int64_t* d, const int64_t* s, const int32_t* dem_off,
                      const int64_t* dem_y, const int64_t* dem_free, const int64_t* flow_off,
                      const int32_t* flow_b, const int64_t* flow_cnt, const int32_t* sup_off,
                      const int64_t* sup_y, const int64_t* sup_free, const int64_t* sup_matched,
                      int32_t which, int64_t* count, char* msgs, int32_t msgs_cap) {
  return guarded([&] {
    const otpr::CopyInstance ci = make_copy(n_a, n_b, k, 0.5, unit_ceil, unit_ceil, d, s);
    otpr::ClusterState st;
    st.demand.resize(n_a);
    st.supply.resize(n_b);
    for (int32_t a = 0; a < n_a; ++a)
      for (int32_t c = dem_off[a]; c < dem_off[a + 1]; ++c) {
        otpr::DemandCluster dc;
        dc.y = dem_y[c];
        dc.free_count = dem_free[c];
        for (int64_t f = flow_off[c]; f < flow_off[c + 1]; ++f) dc.flow.emplace_back(flow_b[f], flow_cnt[f]);
        st.demand[a].push_back(std::move(dc));
      }
    for (int32_t b = 0; b < n_b; ++b)
      for (int32_t c = sup_off[b]; c < sup_off[b + 1]; ++c)
        st.supply[b].push_back(otpr::SupplyCluster{sup_y[c], sup_free[c], sup_matched[c]});
    const otpr::ClusterReport rep =
        which == 0 ? otpr::check_cluster_invariant(st, ci) : otpr::check_cluster_feasibility(st, ci);
    *count = static_cast<int64_t>(rep.violations.size());
    std::string m;
    for (const auto& x : rep.violations) m += (m.empty() ? "" : "\n") + x;
    const size_t n = std::min(m.size(), static_cast<size_t>(msgs_cap - 1));
    std::memcpy(msgs, m.data(), n);
    msgs[n] = 0;
  });
}

}  // extern "C"
