// otprg.hpp — the reference's C++ API (namespace otpr, proj/include/otpr/*.hpp)
// restated in namespace otprg on top of the C ABI (otprg.h).  A caller of
//   otpr::solve_assignment / scale_round_costs / verify_feasibility /
//   matching_cost / gen_uniform_square / solve_ot / sinkhorn
// switches by namespace and links libotprg.so; the types mirror otpr's
// (core.hpp, assignment.hpp, ot.hpp, sinkhorn.hpp) with the same fields,
// semantics and exception classes, so a translation unit can even use both
// libraries side by side (tests/cpp/dropin_test.cpp does).  C++17.
//
// Device path: results equal the reference's threads = 1 results bit for bit
// (the Sinkhorn baseline to a floating-point tolerance), copy mode
// (AssignmentOptions::demand_groups / supply_groups) and the copy/cluster
// solver's primitives and hooks (solve_copy_matching, plan_from_flow,
// ClusterOptions / OTOptions, check_cluster_*) included.
// AssignmentOptions::threads is accepted and ignored (the device path is
// always deterministic).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace otprg {

using Index = std::int32_t;
using DualUnits = std::int64_t;
inline constexpr Index kUnmatched = -1;

// ---- errors (errors.hpp:9-37) ----------------------------------------------
class ParameterError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class InputError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class FormatError : public InputError {
 public:
  using InputError::InputError;
};
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class InvariantViolation : public std::logic_error {
 public:
  using std::logic_error::logic_error;
};
class DeviceError : public std::runtime_error {  // CUDA failures (status 6)
 public:
  using std::runtime_error::runtime_error;
};

// ---- data model (core.hpp) ---------------------------------------------------
template <typename T>
class Matrix {  // dense row-major, rows = demand side A
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols, T fill = T{})
      : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows) * cols, fill) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  T& operator()(Index r, Index c) { return data_[static_cast<std::size_t>(r) * cols_ + c]; }
  const T& operator()(Index r, Index c) const { return data_[static_cast<std::size_t>(r) * cols_ + c]; }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  Matrix transposed() const {
    Matrix t(cols_, rows_);
    for (Index r = 0; r < rows_; ++r)
      for (Index c = 0; c < cols_; ++c) t(c, r) = (*this)(r, c);
    return t;
  }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

struct AssignmentInstance {  // core.hpp:69-81
  Index n_a = 0;
  Index n_b = 0;
  Matrix<double> cost;  // n_a x n_b in [0,1]; empty -> the point sets below
  double norm_factor = 1.0;
  std::uint64_t seed = 0;
  // B200-native extension: 2-D point sets (x, y interleaved) whose cost is
  // gen_uniform_square's sqrt(dx^2+dy^2)/sqrt(2), built on the device.
  std::vector<double> pts_a, pts_b;
  void validate() const;
};

struct ScaledCosts {  // core.hpp:85-96
  double eps = 0.0;
  Matrix<std::int32_t> k;
  std::int32_t unit_floor = 0;
  std::int32_t unit_ceil = 0;
  DualUnits dual_bound() const { return static_cast<DualUnits>(unit_ceil) + 2; }
};

std::int64_t scaled_floor(double c, double eps);
ScaledCosts scale_round_costs(const AssignmentInstance& inst, double eps);

struct DualState {  // core.hpp:109-115
  std::vector<DualUnits> y_a;
  std::vector<DualUnits> y_b;
  DualUnits sum_abs() const;
};

struct Matching {  // core.hpp:117-138
  std::vector<Index> match_of_a;
  std::vector<Index> match_of_b;
  Matching() = default;
  Matching(Index n_a, Index n_b) : match_of_a(n_a, kUnmatched), match_of_b(n_b, kUnmatched) {}
  bool has_a(Index a) const { return match_of_a[a] != kUnmatched; }
  bool has_b(Index b) const { return match_of_b[b] != kUnmatched; }
  void link(Index a, Index b) {
    match_of_a[a] = b;
    match_of_b[b] = a;
  }
  Index size() const;
  void validate() const;
};

double matching_cost(const Matching& m, const AssignmentInstance& inst);

// ---- assignment (assignment.hpp) ---------------------------------------------
struct PhaseWorkset {
  std::vector<Index> b_free;
  std::vector<std::vector<Index>> e_admissible;
  std::vector<Index> a_touched;
  std::vector<std::pair<Index, Index>> m_prime;
  std::vector<Index> a_double;
  std::vector<std::pair<Index, Index>> m_double;
  std::size_t edge_count() const;
};

struct SolveStats {
  int phases = 0;
  std::vector<std::int64_t> free_counts;
  std::int64_t sum_ni = 0;
  DualState duals_final;  // internal orientation (see swapped)
  bool swapped = false;
  bool full_match_termination = false;
  std::int64_t phase_bound(double eps) const;
  std::int64_t sum_ni_bound(double eps, Index n) const;
};

struct PhaseSnapshot {
  int phase;
  const ScaledCosts& costs;
  const DualState& duals;
  const Matching& matching;
  const PhaseWorkset& workset;
  DualUnits sum_abs_before;
  DualUnits sum_abs_after;
};
using PhaseObserver = std::function<void(const PhaseSnapshot&)>;

struct AssignmentOptions {
  double eps = 0.1;
  int threads = 1;
  bool check_invariants = false;
  PhaseObserver observer;
  const std::vector<Index>* demand_groups = nullptr;
  const std::vector<Index>* supply_groups = nullptr;
  int device = 0;   // CUDA device
  int storage = 0;  // otprg_storage (0 = auto)
  // 2-D point instances (cost empty): 0 auto (on the fly when the rounded
  // matrix would not fit in free device memory), 1 matrix, 2 on the fly (the
  // scans round the point costs through the exact threshold table; no kT).
  int costs = 0;
  // Multi-GPU: non-empty = the rows of A are sharded over these
  // CUDA devices (one shard per entry; a device listed several times holds
  // several logical shards) and solved by the device-resident loop
  // (otprg_create_multi / otprg_shard_solve_resident).  Point instances only;
  // results are bit-identical to the single-GPU solve.
  std::vector<int> devices;
  int shard_k = 16;  // candidates per shard and proposer per exchange round
};

struct FeasibilityReport {
  std::vector<std::string> violations;  // the first violation (device suite)
  std::vector<std::string> notes;
  std::int64_t count = 0;  // number of violations
  bool ok() const { return violations.empty(); }
};

FeasibilityReport verify_feasibility(const ScaledCosts& sc, const DualState& duals, const Matching& m);
std::pair<Matching, SolveStats> solve_assignment(const AssignmentInstance& inst,
                                                 const AssignmentOptions& opt);
AssignmentInstance gen_uniform_square(Index n, std::uint64_t seed);  // dense, like the reference

// ---- optimal transport (ot.hpp) ------------------------------------------------
struct OTInstance {
  std::vector<double> mu;
  std::vector<double> nu;
  Matrix<double> cost;
  double norm_factor = 1.0;
  std::uint64_t seed = 0;
  Index n_a() const { return static_cast<Index>(mu.size()); }
  Index n_b() const { return static_cast<Index>(nu.size()); }
};

struct TransportPlan {  // core.hpp:150-162
  struct Entry {
    Index a;
    Index b;
    double mass;
  };
  std::vector<Entry> entries;
  double cost = 0.0;
};

OTInstance gen_random_ot_rational(Index n_a, Index n_b, std::uint64_t seed);

struct ScaledMasses {  // ot.hpp:40-49
  double theta = 0.0;
  std::vector<std::int64_t> d;
  std::vector<std::int64_t> s;
  std::int64_t total_d() const;
  std::int64_t total_s() const;
};
ScaledMasses scale_and_round(const OTInstance& inst, double eps);

struct CopyInstance {  // ot.hpp:52-63
  ScaledCosts costs;
  std::vector<std::int64_t> demand_copies;
  std::vector<std::int64_t> supply_copies;
  std::int64_t total_demand() const;
  std::int64_t total_supply() const;
};

struct DemandCluster {  // ot.hpp:65-75
  DualUnits y = 0;
  std::int64_t free_count = 0;
  std::vector<std::pair<Index, std::int64_t>> flow;  // (b, copies), sorted
  std::int64_t matched() const;
  std::int64_t count() const { return free_count + matched(); }
};

struct SupplyCluster {  // ot.hpp:77-83
  DualUnits y = 0;
  std::int64_t free_count = 0;
  std::int64_t matched_count = 0;
  std::int64_t count() const { return free_count + matched_count; }
};

struct ClusterState {  // ot.hpp:85-95
  std::vector<std::vector<DemandCluster>> demand;
  std::vector<std::vector<SupplyCluster>> supply;
  Matrix<std::int64_t> flow_matrix(Index n_a, Index n_b) const;
  std::int64_t free_supply_total() const;
  std::int64_t free_demand_of(Index a) const;
  DualUnits sum_abs_duals() const;
};

struct ClusterReport {  // ot.hpp:97-100
  std::vector<std::string> violations;
  bool ok() const { return violations.empty(); }
};
ClusterReport check_cluster_invariant(const ClusterState& state, const CopyInstance& inst);
ClusterReport check_cluster_feasibility(const ClusterState& state, const CopyInstance& inst);

struct ClusterPhaseSnapshot {  // ot.hpp:115-122 (valid during the callback)
  int phase;
  const CopyInstance& inst;
  const ClusterState& state;
  std::int64_t n_i;
  DualUnits sum_abs_before;
  DualUnits sum_abs_after;
};

struct ClusterOptions {  // ot.hpp:124-129
  bool check_invariants = false;
  std::function<void(const ClusterPhaseSnapshot&)> observer;
};

struct ClusterSolveResult {  // ot.hpp:131-135
  ClusterState state;
  Matrix<std::int64_t> flow;
  SolveStats stats;
};

ClusterSolveResult solve_copy_matching(const CopyInstance& inst, double eps,
                                       const ClusterOptions& opt = {});
TransportPlan plan_from_flow(const Matrix<std::int64_t>& flow, const ScaledMasses& sm,
                             const OTInstance& inst);

struct OTOptions {  // ot.hpp:153-156
  bool check_invariants = false;
  std::function<void(const ClusterPhaseSnapshot&)> observer;
};
std::pair<TransportPlan, SolveStats> solve_ot(const OTInstance& inst, double eps,
                                              const OTOptions& opt = {});

// ---- Sinkhorn baseline (sinkhorn.hpp) ---------------------------------------------
struct SinkhornConfig {
  double reg = 0.01;
  int max_iters = 10000;
  double tol = 1e-9;
  double time_budget_ms = 0.0;
};
struct SinkhornResult {
  TransportPlan plan;
  int iters = 0;
  double cost = 0.0;
  bool converged = false;
  double marginal_violation = 0.0;
};
SinkhornResult sinkhorn(const OTInstance& inst, const SinkhornConfig& cfg);

}  // namespace otprg
