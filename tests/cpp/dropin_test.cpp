// dropin_test.cpp — the C++ drop-in check: the same calls against the
// UNMODIFIED reference (namespace otpr, oracle/_ref/libotpr_ref.so) and
// against this library (namespace otprg, libotprg.so), side by side in one
// program, results compared field by field.  Needs a GPU (run by
// tests/test_gpu_cpp_dropin.py).  Built by tests/cpp/Makefile (needs the
// reference headers, i.e. the build container).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "otpr/assignment.hpp"
#include "otpr/core.hpp"
#include "otpr/instances.hpp"
#include "otpr/ot.hpp"
#include "otpr/sinkhorn.hpp"
#include "otprg.hpp"

static int g_fail = 0;
#define EXPECT(cond, what)                                       \
  do {                                                           \
    if (!(cond)) {                                               \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++g_fail;                                                  \
    }                                                            \
  } while (0)

static otprg::AssignmentInstance to_g(const otpr::AssignmentInstance& r) {
  otprg::AssignmentInstance g;
  g.n_a = r.n_a;
  g.n_b = r.n_b;
  g.cost = otprg::Matrix<double>(r.n_a, r.n_b);
  std::memcpy(g.cost.data(), r.cost.data(), r.cost.size() * sizeof(double));
  g.norm_factor = r.norm_factor;
  g.seed = r.seed;
  return g;
}

static otpr::AssignmentInstance random_instance(int n_a, int n_b, uint64_t seed) {  // test_util.hpp
  std::mt19937_64 rng(seed);
  otpr::AssignmentInstance inst;
  inst.n_a = n_a;
  inst.n_b = n_b;
  inst.cost = otpr::Matrix<double>(n_a, n_b);
  for (int a = 0; a < n_a; ++a)
    for (int b = 0; b < n_b; ++b) inst.cost(a, b) = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return inst;
}

template <typename MR, typename SR, typename MG, typename SG>
static void same_result(const MR& mr, const SR& sr, const MG& mg, const SG& sg, const char* name) {
  EXPECT(mr.match_of_a == mg.match_of_a, name);
  EXPECT(mr.match_of_b == mg.match_of_b, name);
  EXPECT(sr.phases == sg.phases, name);
  EXPECT(sr.free_counts == sg.free_counts, name);
  EXPECT(sr.sum_ni == sg.sum_ni, name);
  EXPECT(sr.duals_final.y_a == sg.duals_final.y_a, name);
  EXPECT(sr.duals_final.y_b == sg.duals_final.y_b, name);
  EXPECT(sr.swapped == sg.swapped, name);
  EXPECT(sr.full_match_termination == sg.full_match_termination, name);
}

static void assignment_cases() {
  for (uint64_t seed : {1, 2, 3}) {
    const otpr::AssignmentInstance r = otpr::gen_uniform_square(1000, seed);
    otpr::AssignmentOptions ro;
    ro.eps = 0.01;
    auto [mr, sr] = otpr::solve_assignment(r, ro);
    otprg::AssignmentOptions go;
    go.eps = 0.01;
    const otprg::AssignmentInstance g = to_g(r);
    auto [mg, sg] = otprg::solve_assignment(g, go);
    same_result(mr, sr, mg, sg, "square dense");
    EXPECT(otpr::matching_cost(mr, r) == otprg::matching_cost(mg, g), "matching_cost bits");
    // the point-set form (cost built on the device)
    otprg::AssignmentInstance gp = otprg::gen_uniform_square(1000, seed);
    gp.cost = otprg::Matrix<double>();
    auto [mp, sp] = otprg::solve_assignment(gp, go);
    same_result(mr, sr, mp, sp, "square points");
    EXPECT(otpr::matching_cost(mr, r) == otprg::matching_cost(mp, gp), "points matching_cost bits");
    // costs on the fly (no rounded matrix anywhere; threshold table)
    otprg::AssignmentOptions gf = go;
    gf.costs = 2;
    auto [mf, sf] = otprg::solve_assignment(gp, gf);
    same_result(mr, sr, mf, sf, "square points, costs on the fly");
    // A rows sharded over several (logical) devices: the resident multi-GPU loop
    for (int G : {1, 3}) {
      otprg::AssignmentOptions gm = go;
      gm.devices.assign(G, 0);
      auto [mm, sm] = otprg::solve_assignment(gp, gm);
      same_result(mr, sr, mm, sm, G == 1 ? "sharded, 1 device" : "sharded, 3 logical devices");
      gm.costs = 2;
      auto [mo, so] = otprg::solve_assignment(gp, gm);
      same_result(mr, sr, mo, so, "sharded on the fly");
    }
  }
  for (auto [na, nb] : {std::pair{300, 170}, std::pair{170, 300}}) {
    const otpr::AssignmentInstance r = random_instance(na, nb, 40 + na);
    otpr::AssignmentOptions ro;
    ro.eps = 0.03;
    otprg::AssignmentOptions go;
    go.eps = 0.03;
    auto [mr, sr] = otpr::solve_assignment(r, ro);
    auto [mg, sg] = otprg::solve_assignment(to_g(r), go);
    same_result(mr, sr, mg, sg, "rectangular");
  }
  // rounding
  {
    const otpr::AssignmentInstance r = random_instance(200, 150, 9);
    const auto kr = otpr::scale_round_costs(r, 0.007);
    const auto kg = otprg::scale_round_costs(to_g(r), 0.007);
    EXPECT(kr.unit_floor == kg.unit_floor && kr.unit_ceil == kg.unit_ceil, "units");
    EXPECT(std::memcmp(kr.k.data(), kg.k.data(), kr.k.size() * 4) == 0, "rounded costs");
    EXPECT(otpr::scaled_floor(0.57, 0.1) == otprg::scaled_floor(0.57, 0.1), "scaled_floor");
  }
  // errors
  {
    const otpr::AssignmentInstance r = random_instance(4, 4, 1);
    otprg::AssignmentOptions go;
    go.eps = 1.0;
    bool thrown = false;
    try {
      otprg::solve_assignment(to_g(r), go);
    } catch (const otprg::ParameterError&) {
      thrown = true;
    }
    EXPECT(thrown, "eps = 1 -> ParameterError");
  }
}

struct PhaseRec {
  int phase;
  std::vector<otpr::Index> b_free, m_prime_a, m_prime_b, a_double, a_touched;
  std::vector<std::vector<otpr::Index>> e_admissible;
  std::vector<otpr::DualUnits> y_a, y_b;
  otpr::DualUnits before, after;
};

static void observer_cases() {
  for (uint64_t seed : {131, 262}) {
    const otpr::AssignmentInstance r = random_instance(30, 30, seed);
    std::vector<PhaseRec> ref;
    otpr::AssignmentOptions ro;
    ro.eps = 0.08;
    ro.check_invariants = true;
    ro.observer = [&](const otpr::PhaseSnapshot& s) {
      PhaseRec p{s.phase, s.workset.b_free, {}, {}, s.workset.a_double, s.workset.a_touched,
                 s.workset.e_admissible, s.duals.y_a, s.duals.y_b, s.sum_abs_before, s.sum_abs_after};
      for (auto [a, b] : s.workset.m_prime) {
        p.m_prime_a.push_back(a);
        p.m_prime_b.push_back(b);
      }
      ref.push_back(std::move(p));
    };
    auto [mr, sr] = otpr::solve_assignment(r, ro);
    size_t i = 0;
    otprg::AssignmentOptions go;
    go.eps = 0.08;
    go.check_invariants = true;
    go.observer = [&](const otprg::PhaseSnapshot& s) {
      if (i >= ref.size()) {
        EXPECT(false, "more phases than the reference");
        return;
      }
      const PhaseRec& p = ref[i++];
      EXPECT(p.phase == s.phase, "phase");
      EXPECT(p.b_free == s.workset.b_free, "B'");
      EXPECT(p.e_admissible == s.workset.e_admissible, "E'");
      EXPECT(p.a_touched == s.workset.a_touched, "A'");
      EXPECT(p.a_double == s.workset.a_double, "A''");
      std::vector<otpr::Index> ma, mb;
      for (auto [a, b] : s.workset.m_prime) {
        ma.push_back(a);
        mb.push_back(b);
      }
      EXPECT(p.m_prime_a == ma && p.m_prime_b == mb, "M'");
      EXPECT(p.y_a == s.duals.y_a && p.y_b == s.duals.y_b, "duals");
      EXPECT(p.before == s.sum_abs_before && p.after == s.sum_abs_after, "sum_abs");
    };
    auto [mg, sg] = otprg::solve_assignment(to_g(r), go);
    EXPECT(i == ref.size(), "phase count seen by the observer");
    same_result(mr, sr, mg, sg, "observer run");
  }
  // verify_feasibility on a corrupted state: same first message and count
  const otpr::AssignmentInstance r = random_instance(4, 4, 9);
  const auto sc = otpr::scale_round_costs(r, 0.2);
  auto [m, d] = otpr::init_state(sc);
  d.y_b[2] += 10;
  const auto rr = otpr::verify_feasibility(sc, d, m);
  otprg::ScaledCosts gsc;
  gsc.eps = sc.eps;
  gsc.unit_floor = sc.unit_floor;
  gsc.unit_ceil = sc.unit_ceil;
  gsc.k = otprg::Matrix<std::int32_t>(4, 4);
  std::memcpy(gsc.k.data(), sc.k.data(), 16 * 4);
  otprg::DualState gd{d.y_a, d.y_b};
  otprg::Matching gm(4, 4);
  const auto gr = otprg::verify_feasibility(gsc, gd, gm);
  EXPECT(!rr.ok() && !gr.ok(), "violations found");
  EXPECT(rr.violations.front() == gr.violations.front(), "first violation message");
  EXPECT(static_cast<int64_t>(rr.violations.size()) == gr.count, "violation count");
}

static void ot_cases() {
  const otpr::OTInstance r = otpr::gen_random_ot_rational(300, 200, 3);
  otprg::OTInstance g;
  g.mu = r.mu;
  g.nu = r.nu;
  g.cost = otprg::Matrix<double>(300, 200);
  std::memcpy(g.cost.data(), r.cost.data(), r.cost.size() * sizeof(double));
  auto [pr, sr] = otpr::solve_ot(r, 0.01);
  auto [pg, sg] = otprg::solve_ot(g, 0.01);
  EXPECT(pr.cost == pg.cost, "OT cost bits");
  EXPECT(pr.entries.size() == pg.entries.size(), "OT entry count");
  bool same = pr.entries.size() == pg.entries.size();
  for (size_t i = 0; same && i < pr.entries.size(); ++i)
    same = pr.entries[i].a == pg.entries[i].a && pr.entries[i].b == pg.entries[i].b &&
           pr.entries[i].mass == pg.entries[i].mass;
  EXPECT(same, "OT plan entries");
  EXPECT(sr.phases == sg.phases && sr.free_counts == sg.free_counts, "OT phases");
  otpr::SinkhornConfig rc;
  rc.reg = 0.05;
  otprg::SinkhornConfig gc;
  gc.reg = 0.05;
  const auto kr = otpr::sinkhorn(r, rc);
  const auto kg = otprg::sinkhorn(g, gc);
  EXPECT(std::abs(kr.iters - kg.iters) <= 1, "sinkhorn iterations");
  EXPECT(std::abs(kr.cost - kg.cost) <= 1e-9 * std::abs(kr.cost), "sinkhorn cost");
}

// copy mode (demand/supply groups, assignment.cpp:81-103, :241-250) with the
// observer: per-phase worksets in the grouped scan order must match.
static void copy_mode_cases() {
  const int d_copies[4] = {3, 2, 4, 1}, s_copies[3] = {2, 3, 4};
  const otpr::AssignmentInstance orig = random_instance(4, 3, 11);
  std::vector<otpr::Index> dg, sg;
  for (int a = 0; a < 4; ++a)
    for (int c = 0; c < d_copies[a]; ++c) dg.push_back(a);
  for (int b = 0; b < 3; ++b)
    for (int c = 0; c < s_copies[b]; ++c) sg.push_back(b);
  otpr::AssignmentInstance r;
  r.n_a = static_cast<int>(dg.size());
  r.n_b = static_cast<int>(sg.size());
  r.cost = otpr::Matrix<double>(r.n_a, r.n_b);
  for (int i = 0; i < r.n_a; ++i)
    for (int j = 0; j < r.n_b; ++j) r.cost(i, j) = orig.cost(dg[i], sg[j]);
  for (double eps : {0.2, 0.1}) {
    std::vector<std::vector<std::vector<otpr::Index>>> ref_e;
    std::vector<std::vector<otpr::Index>> ref_mb;
    otpr::AssignmentOptions ro;
    ro.eps = eps;
    ro.demand_groups = &dg;
    ro.supply_groups = &sg;
    ro.check_invariants = true;
    ro.observer = [&](const otpr::PhaseSnapshot& s) {
      ref_e.push_back(s.workset.e_admissible);
      ref_mb.push_back(s.matching.match_of_b);
    };
    auto [mr, sr] = otpr::solve_assignment(r, ro);
    size_t i = 0;
    otprg::AssignmentOptions go;
    go.eps = eps;
    go.demand_groups = &dg;
    go.supply_groups = &sg;
    go.check_invariants = true;
    go.observer = [&](const otprg::PhaseSnapshot& s) {
      if (i < ref_e.size()) {
        EXPECT(ref_e[i] == s.workset.e_admissible, "copy-mode E' (grouped order)");
        EXPECT(ref_mb[i] == s.matching.match_of_b, "copy-mode matching");
      }
      ++i;
    };
    auto [mg, sg2] = otprg::solve_assignment(to_g(r), go);
    EXPECT(i == ref_e.size(), "copy-mode phase count");
    same_result(mr, sr, mg, sg2, "copy mode");
  }
}

// copy/cluster solver primitives (ot.hpp:97-156): solve_copy_matching with
// check_invariants and an observer (flow after every phase), the final state,
// check_cluster_* on it, plan_from_flow, and solve_ot with OTOptions.
static void cluster_cases() {
  std::mt19937_64 rng(777);
  for (int trial = 0; trial < 12; ++trial) {
    const double eps = 0.1 + 0.05 * static_cast<double>(rng() % 5);
    const int n_a = static_cast<int>(rng() % 5) + 2, n_b = static_cast<int>(rng() % 5) + 2;
    const otpr::AssignmentInstance orig = random_instance(n_a, n_b, rng());
    otpr::CopyInstance rc;
    rc.costs = otpr::scale_round_costs(orig, eps);
    std::int64_t td = 0, ts = 0;
    for (int a = 0; a < n_a; ++a) rc.demand_copies.push_back(static_cast<std::int64_t>(rng() % 12) + 1), td += rc.demand_copies.back();
    for (int b = 0; b < n_b; ++b) {
      const std::int64_t room = td - ts;
      rc.supply_copies.push_back(room > 0 ? static_cast<std::int64_t>(rng() % (room + 1)) : 0);
      ts += rc.supply_copies.back();
    }
    otprg::CopyInstance gc;
    gc.costs.eps = rc.costs.eps;
    gc.costs.unit_floor = rc.costs.unit_floor;
    gc.costs.unit_ceil = rc.costs.unit_ceil;
    gc.costs.k = otprg::Matrix<std::int32_t>(n_a, n_b);
    std::memcpy(gc.costs.k.data(), rc.costs.k.data(), rc.costs.k.size() * 4);
    gc.demand_copies = rc.demand_copies;
    gc.supply_copies = rc.supply_copies;
    std::vector<std::vector<std::int64_t>> rflows, gflows;
    otpr::ClusterOptions ro;
    ro.check_invariants = true;
    ro.observer = [&](const otpr::ClusterPhaseSnapshot& sn) {
      const auto f = sn.state.flow_matrix(n_a, n_b);
      rflows.emplace_back(f.data(), f.data() + f.size());
    };
    otprg::ClusterOptions go;
    go.check_invariants = true;
    go.observer = [&](const otprg::ClusterPhaseSnapshot& sn) {
      const auto f = sn.state.flow_matrix(n_a, n_b);
      gflows.emplace_back(f.data(), f.data() + f.size());
    };
    const auto rr = otpr::solve_copy_matching(rc, eps, ro);
    const auto gr = otprg::solve_copy_matching(gc, eps, go);
    EXPECT(rr.stats.phases == gr.stats.phases && rr.stats.free_counts == gr.stats.free_counts, "copy matching phases");
    EXPECT(rflows == gflows, "copy matching flow after every phase");
    EXPECT(std::memcmp(rr.flow.data(), gr.flow.data(), rr.flow.size() * 8) == 0, "copy matching final flow");
    bool same_state = rr.state.demand.size() == gr.state.demand.size();
    for (size_t a = 0; same_state && a < rr.state.demand.size(); ++a) {
      same_state = rr.state.demand[a].size() == gr.state.demand[a].size();
      for (size_t c = 0; same_state && c < rr.state.demand[a].size(); ++c)
        same_state = rr.state.demand[a][c].y == gr.state.demand[a][c].y &&
                     rr.state.demand[a][c].free_count == gr.state.demand[a][c].free_count &&
                     rr.state.demand[a][c].flow == gr.state.demand[a][c].flow;
    }
    for (size_t b = 0; same_state && b < rr.state.supply.size(); ++b) {
      same_state = rr.state.supply[b].size() == gr.state.supply[b].size();
      for (size_t c = 0; same_state && c < rr.state.supply[b].size(); ++c)
        same_state = rr.state.supply[b][c].y == gr.state.supply[b][c].y &&
                     rr.state.supply[b][c].free_count == gr.state.supply[b][c].free_count &&
                     rr.state.supply[b][c].matched_count == gr.state.supply[b][c].matched_count;
    }
    EXPECT(same_state, "copy matching final ClusterState");
    EXPECT(otprg::check_cluster_invariant(gr.state, gc).ok() && otprg::check_cluster_feasibility(gr.state, gc).ok(),
           "cluster checks pass on the final state");
    // a corrupted state: the same violation list as the reference
    otpr::ClusterState rbad = rr.state;
    otprg::ClusterState gbad = gr.state;
    if (!rbad.supply.empty() && !rbad.supply[0].empty()) {
      rbad.supply[0][0].y += 3;
      gbad.supply[0][0].y += 3;
    }
    EXPECT(otpr::check_cluster_invariant(rbad, rc).violations == otprg::check_cluster_invariant(gbad, gc).violations,
           "cluster invariant messages");
    EXPECT(otpr::check_cluster_feasibility(rbad, rc).violations ==
               otprg::check_cluster_feasibility(gbad, gc).violations,
           "cluster feasibility messages");
  }
  // solve_ot = scale_and_round -> solve_copy_matching(eps/3) -> plan_from_flow, with hooks
  const otpr::OTInstance r = otpr::gen_random_ot_rational(40, 30, 9);
  otprg::OTInstance g;
  g.mu = r.mu;
  g.nu = r.nu;
  g.cost = otprg::Matrix<double>(40, 30);
  std::memcpy(g.cost.data(), r.cost.data(), r.cost.size() * sizeof(double));
  int phases_seen = 0;
  otprg::OTOptions oo;
  oo.check_invariants = true;
  oo.observer = [&](const otprg::ClusterPhaseSnapshot& sn) { phases_seen = sn.phase; };
  auto [pr, sr] = otpr::solve_ot(r, 0.1);
  auto [pg, sg] = otprg::solve_ot(g, 0.1, oo);
  EXPECT(pr.cost == pg.cost && sr.free_counts == sg.free_counts, "solve_ot with OTOptions");
  EXPECT(phases_seen == sg.phases, "OT observer saw every phase");
  const auto smg = otprg::scale_and_round(g, 0.1 / 3.0);
  const auto smr = otpr::scale_and_round(r, 0.1 / 3.0);
  EXPECT(smg.d == smr.d && smg.s == smr.s && smg.theta == smr.theta, "scale_and_round");
  otpr::CopyInstance rc;
  rc.costs = otpr::scale_round_costs(otpr::AssignmentInstance{40, 30, r.cost}, 0.1 / 3.0);
  rc.demand_copies = smr.d;
  rc.supply_copies = smr.s;
  const auto rr = otpr::solve_copy_matching(rc, 0.1 / 3.0);
  otprg::Matrix<std::int64_t> gf(40, 30);
  std::memcpy(gf.data(), rr.flow.data(), rr.flow.size() * 8);
  const auto plan = otprg::plan_from_flow(gf, smg, g);
  EXPECT(plan.cost == pr.cost && plan.entries.size() == pr.entries.size(), "plan_from_flow");
}

int main() {
  assignment_cases();
  observer_cases();
  ot_cases();
  copy_mode_cases();
  cluster_cases();
  if (g_fail) {
    std::printf("dropin: %d failures\n", g_fail);
    return 1;
  }
  std::printf("dropin: all checks passed\n");
  return 0;
}
