"""ctypes binding of libotprg.so (the C ABI in include/otprg.h).

The shared library is built in-tree (paper_2203_03732_b200/lib/libotprg.so)
by ``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2203_03732_b200/csrc``.  There is no fallback: if the library
is missing, importing the solver raises instead of silently computing on the
CPU.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", os.environ.get("OTPRG_LIB", "libotprg.so"))
CSRC = os.path.join(PKG_DIR, "csrc")

OK, PARAMETER, INPUT, NUMERICAL, INVARIANT, DEVICE, ABORTED = 0, 2, 3, 4, 5, 6, 7
IPC_HANDLE_BYTES = 64  # OTPRG_IPC_HANDLE_BYTES
COST_DENSE_F64, COST_POINTS2D, COST_L1_U8 = 0, 1, 2
STORAGE = {"auto": 0, "u8": 1, "u16": 2, "u32": 3}
MAX_PHASES = 1 << 24  # OTPRG_MAX_PHASES
FLAG_ON_THE_FLY = 1  # OTPRG_FLAG_ON_THE_FLY


class Problem(C.Structure):
    _fields_ = [
        ("n_a", C.c_int32), ("n_b", C.c_int32), ("eps", C.c_double),
        ("cost_kind", C.c_int32), ("storage", C.c_int32),
        ("cost", C.c_void_p), ("pts_a", C.c_void_p), ("pts_b", C.c_void_p),
        ("img_a", C.c_void_p), ("img_b", C.c_void_p),
        ("dim", C.c_int32), ("flags", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("match_of_a", C.c_void_p), ("match_of_b", C.c_void_p),
        ("y_a", C.c_void_p), ("y_b", C.c_void_p),
        ("free_counts", C.c_void_p), ("free_cap", C.c_int64),
        ("phases", C.c_int64), ("sum_ni", C.c_int64),
        ("swapped", C.c_int32), ("full_match_termination", C.c_int32),
        ("cost", C.c_double),
        ("build_ms", C.c_double), ("solve_ms", C.c_double), ("phase1_ms", C.c_double),
        ("loop_ms", C.c_double), ("solve_d2h_ms", C.c_double),
        ("bytes_touched", C.c_int64), ("bytes_alg", C.c_int64),
        ("width", C.c_int32), ("gpu_launches", C.c_int32),
        ("chain_stats", C.c_int64 * 8),
        ("refill_rounds", C.c_int32), ("n_shards", C.c_int32),
    ]


class Feasibility(C.Structure):
    _fields_ = [
        ("violations", C.c_int64), ("kind", C.c_int32), ("a", C.c_int32), ("b", C.c_int32),
        ("pad", C.c_int32), ("sum", C.c_int64), ("k", C.c_int64),
    ]


class CopyInstance(C.Structure):
    _fields_ = [("n_a", C.c_int32), ("n_b", C.c_int32), ("k", C.c_void_p), ("unit_ceil", C.c_int64),
                ("demand_copies", C.c_void_p), ("supply_copies", C.c_void_p)]


class ClusterState(C.Structure):
    _fields_ = [("n_a", C.c_int32), ("n_b", C.c_int32), ("dem_off", C.c_void_p),
                ("dem_y", C.c_void_p), ("dem_free", C.c_void_p), ("flow_off", C.c_void_p),
                ("flow_b", C.c_void_p), ("flow_cnt", C.c_void_p), ("sup_off", C.c_void_p),
                ("sup_y", C.c_void_p), ("sup_free", C.c_void_p), ("sup_matched", C.c_void_p)]


class ClusterSnapshot(C.Structure):
    _fields_ = [("phase", C.c_int64), ("n_i", C.c_int64), ("sum_abs_before", C.c_int64),
                ("sum_abs_after", C.c_int64), ("inst", CopyInstance), ("state", ClusterState)]


CLUSTER_OBSERVER = C.CFUNCTYPE(C.c_int, C.POINTER(ClusterSnapshot), C.c_void_p)


class OTOptions(C.Structure):
    _fields_ = [("check_invariants", C.c_int32), ("pad", C.c_int32),
                ("observer", CLUSTER_OBSERVER), ("user", C.c_void_p)]


class CopyResult(C.Structure):
    _fields_ = [("flow", C.c_void_p), ("free_counts", C.c_void_p), ("free_cap", C.c_int64),
                ("phases", C.c_int64), ("sum_ni", C.c_int64), ("full_match_termination", C.c_int32),
                ("gpu_launches", C.c_int32)]


EXPORTS = [
    "otprg_create", "otprg_destroy", "otprg_last_error", "otprg_version", "otprg_scaled_floor",
    "otprg_solve_assignment", "otprg_prepare", "otprg_solve_prepared", "otprg_scale_round_costs",
    "otprg_uniform_square_points", "otprg_flush_l2", "otprg_begin", "otprg_step",
    "otprg_snapshot", "otprg_finish", "otprg_timer_start", "otprg_timer_stop",
    "otprg_set_trace", "otprg_get_trace", "otprg_load_mnist_pair", "otprg_solve_ot",
    "otprg_ot_scale_and_round", "otprg_random_ot_rational", "otprg_shard_prepare",
    "otprg_shard_begin", "otprg_shard_top", "otprg_shard_scan", "otprg_shard_da",
    "otprg_shard_finish", "otprg_set_stream", "otprg_sinkhorn", "otprg_groups_begin",
    "otprg_groups_step", "otprg_groups_finish", "otprg_verify_feasibility", "otprg_verify_host", "otprg_admissible",
    "otprg_solve_ot_opts", "otprg_solve_copy_matching", "otprg_copy_state",
    "otprg_check_cluster_state", "otprg_plan_from_flow", "otprg_points_threshold_table",
    "otprg_mem_info", "otprg_verify_result", "otprg_create_multi", "otprg_set_shard_k",
    "otprg_shard_solve_resident", "otprg_shard_ipc_export", "otprg_shard_ipc_attach",
    "otprg_selftest_exchange",
]

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    """Load libotprg.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.otprg_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.otprg_destroy.argtypes = [vp]
    L.otprg_destroy.restype = None
    L.otprg_last_error.argtypes = [vp]
    L.otprg_last_error.restype = C.c_char_p
    L.otprg_scaled_floor.argtypes = [C.c_double, C.c_double]
    L.otprg_scaled_floor.restype = C.c_int64
    for fn in ("otprg_solve_assignment", "otprg_prepare"):
        getattr(L, fn).argtypes = [vp, C.POINTER(Problem), C.POINTER(Result)]
    L.otprg_solve_prepared.argtypes = [vp, C.POINTER(Result)]
    L.otprg_scale_round_costs.argtypes = [vp, C.POINTER(Problem), vp, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32)]
    L.otprg_uniform_square_points.argtypes = [C.c_int32, C.c_uint64, vp, vp]
    L.otprg_flush_l2.argtypes = [vp]
    L.otprg_mem_info.argtypes = [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.otprg_begin.argtypes = [vp]
    L.otprg_step.argtypes = [vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.otprg_snapshot.argtypes = [vp, C.POINTER(Result)]
    L.otprg_finish.argtypes = [vp, C.POINTER(Result)]
    L.otprg_timer_start.argtypes = [vp]
    L.otprg_timer_stop.argtypes = [vp, C.POINTER(C.c_double)]
    L.otprg_set_trace.argtypes = [vp, C.c_int64]
    L.otprg_get_trace.argtypes = [vp, vp, C.c_int64]
    L.otprg_load_mnist_pair.argtypes = [C.c_char_p, C.c_int32, C.c_uint64, vp, vp, C.c_char_p,
                                        C.c_int32]
    L.otprg_solve_ot.argtypes = [vp, vp, vp]
    L.otprg_points_threshold_table.restype = C.c_int32
    L.otprg_points_threshold_table.argtypes = [C.c_double, vp, C.c_int32]
    L.otprg_solve_ot_opts.argtypes = [vp, vp, C.POINTER(OTOptions), vp]
    L.otprg_solve_copy_matching.argtypes = [vp, C.POINTER(CopyInstance), C.c_double,
                                            C.POINTER(OTOptions), C.POINTER(CopyResult)]
    L.otprg_copy_state.argtypes = [vp, C.POINTER(ClusterState)]
    L.otprg_check_cluster_state.argtypes = [C.POINTER(ClusterState), C.POINTER(CopyInstance),
                                            C.c_int32, C.POINTER(C.c_int64), C.c_char_p, C.c_int32]
    L.otprg_plan_from_flow.argtypes = [vp, vp, C.c_double, vp, vp, vp]
    L.otprg_ot_scale_and_round.argtypes = [C.c_int32, C.c_int32, vp, vp, C.c_double, vp, vp,
                                           C.POINTER(C.c_double)]
    L.otprg_random_ot_rational.argtypes = [C.c_int32, C.c_int32, C.c_uint64, vp, vp, vp]
    L.otprg_shard_prepare.argtypes = [vp, C.POINTER(Problem), C.c_int32, C.c_int32, C.c_int32, vp]
    L.otprg_shard_begin.argtypes = [vp]
    L.otprg_create_multi.argtypes = [vp, C.c_int32, C.POINTER(vp)]
    L.otprg_set_shard_k.argtypes = [vp, C.c_int32]
    L.otprg_shard_solve_resident.argtypes = [vp, C.c_int32, C.POINTER(Result)]
    L.otprg_shard_ipc_export.argtypes = [vp, C.c_int32, C.c_int32, vp]
    L.otprg_shard_ipc_attach.argtypes = [vp, vp, C.c_int32, vp]
    L.otprg_selftest_exchange.argtypes = [C.c_int32] * 6 + [C.POINTER(C.c_int64)]
    L.otprg_shard_top.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.otprg_shard_scan.argtypes = [vp, vp, vp, C.c_int32, C.c_int32]
    L.otprg_shard_da.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
    L.otprg_shard_finish.argtypes = [vp, C.POINTER(Result)]
    L.otprg_set_stream.argtypes = [vp, vp]
    L.otprg_groups_begin.argtypes = [vp, C.POINTER(Problem), vp, vp]
    L.otprg_groups_step.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    L.otprg_groups_finish.argtypes = [vp, C.POINTER(Result)]
    L.otprg_sinkhorn.argtypes = [vp, vp, vp, vp]
    L.otprg_verify_feasibility.argtypes = [vp, C.POINTER(Feasibility)]
    L.otprg_verify_host.argtypes = [vp, C.c_int32, C.c_int32, vp, C.c_int32, vp, vp, vp, vp,
                                    C.POINTER(Feasibility)]
    L.otprg_verify_result.argtypes = [vp, vp, vp, vp, vp, C.POINTER(Feasibility)]
    L.otprg_admissible.argtypes = [vp, vp, vp, vp, C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]
    _lib = L
    return L


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data
