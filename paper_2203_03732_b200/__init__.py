"""paper_2203_03732_b200 — B200-native push-relabel eps-approximate assignment
solver (arXiv 2203.03732), a drop-in for the reference ``otpr`` assignment
path.  See DESIGN.md for the device design and INTEGRATION.md for the C ABI.
"""
from .api import (  # noqa: F401
    AssignmentInstance, AssignmentOptions, DeviceError, DualState, FormatError, InputError,
    InvariantViolation, Matching, NumericalError, ParameterError, ScaledCosts, SolveStats, Solver,
    gen_uniform_square, get_solver, l1_cost, load_mnist_pair, matching_cost, points_cost,
    scale_round_costs, scaled_floor, solve_assignment, OTInstance, TransportPlan, ScaledMasses,
    gen_random_ot_rational, scale_and_round, solve_ot, FeasibilityReport, PhaseSnapshot,
    PhaseWorkset, verify_feasibility, SinkhornConfig, SinkhornResult, sinkhorn, reg_for_eps,
    CopyInstance, DemandCluster, SupplyCluster, ClusterState, ClusterReport, ClusterPhaseSnapshot,
    ClusterOptions, OTOptions, ClusterSolveResult, check_cluster_invariant, check_cluster_feasibility,
    solve_copy_matching, plan_from_flow, last_cluster_state,
)

__all__ = [
    "AssignmentInstance", "AssignmentOptions", "DeviceError", "DualState", "FormatError",
    "InputError", "InvariantViolation", "Matching", "NumericalError", "ParameterError",
    "ScaledCosts", "SolveStats", "Solver", "gen_uniform_square", "get_solver", "l1_cost",
    "load_mnist_pair", "matching_cost", "points_cost", "scale_round_costs", "scaled_floor",
    "solve_assignment", "OTInstance", "TransportPlan", "ScaledMasses", "gen_random_ot_rational",
    "scale_and_round", "solve_ot", "FeasibilityReport", "PhaseSnapshot", "PhaseWorkset",
    "verify_feasibility", "SinkhornConfig", "SinkhornResult", "sinkhorn", "reg_for_eps",
    "CopyInstance", "DemandCluster", "SupplyCluster", "ClusterState", "ClusterReport",
    "ClusterPhaseSnapshot", "ClusterOptions", "OTOptions", "ClusterSolveResult",
    "check_cluster_invariant", "check_cluster_feasibility", "solve_copy_matching", "plan_from_flow",
    "last_cluster_state",
]
