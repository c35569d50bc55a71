"""ctypes access to the parity checkers — TEST INFRASTRUCTURE ONLY.

* ``Oracle``  -> oracle/liboracle.so, our plain-C restatement of the reference
  assignment path (oracle/otpr_oracle.c; each function cites the reference
  file:line it follows).
* ``Reference`` -> oracle/_ref/libotpr_ref.so, the unmodified reference library
  built from /root/reference/proj/src by oracle/Makefile, wrapped by
  oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this module.  The product package
(paper_2203_03732_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libotpr_ref.so")
REF_DIR = os.environ.get("OTPR_REF_DIR", "/root/reference/proj")

FNV_OFFSET = 0xCBF29CE484222325

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def fnv1a64(arr: np.ndarray, h: int = FNV_OFFSET) -> int:
    """FNV-1a-64 over the little-endian bytes of ``arr``."""
    data = np.ascontiguousarray(arr).view(np.uint8)
    # vectorised in chunks would change nothing semantically; plain loop in C
    lib = Oracle.get()
    return int(lib.lib.orc_fnv1a64(data.ctypes.data_as(C.c_void_p), data.size, C.c_uint64(h)))


def build(ref: bool = True) -> None:
    """Compile liboracle.so (always) and _ref/libotpr_ref.so (when the reference tree exists)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_DIR):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


@dataclass
class AssignResult:
    match_of_a: np.ndarray
    match_of_b: np.ndarray
    y_a: np.ndarray
    y_b: np.ndarray
    free_counts: np.ndarray
    phases: int
    sum_ni: int
    swapped: bool
    full_match_termination: bool
    cost: float
    solve_ms: float = 0.0
    round_ms: float = 0.0
    extra: dict = field(default_factory=dict)

    def pins(self) -> dict:
        """The SURVEY.md §8(c) golden-pin tuple for this result."""
        return {
            "phases": int(self.phases),
            "sum_ni": int(self.sum_ni),
            "cost_hex": float(self.cost).hex(),
            "fnv_match": "%016x" % fnv1a64(self.match_of_a.astype(np.int32)),
            "fnv_duals": "%016x" % fnv1a64(np.concatenate([self.y_a, self.y_b]).astype(np.int64)),
            "fnv_free": "%016x" % fnv1a64(self.free_counts.astype(np.int64)),
        }


class _OrcStats(C.Structure):
    _fields_ = [("phases", C.c_int64), ("sum_ni", C.c_int64), ("swapped", C.c_int32),
                ("full_match_termination", C.c_int32), ("cost", C.c_double)]


class _RefStats(C.Structure):
    _fields_ = [("phases", C.c_int64), ("sum_ni", C.c_int64), ("swapped", C.c_int32),
                ("full_match_termination", C.c_int32), ("cost", C.c_double),
                ("solve_ms", C.c_double), ("round_ms", C.c_double),
                ("n_free_counts", C.c_int64)]


class _RefOtStats(C.Structure):
    _fields_ = [("phases", C.c_int64), ("sum_ni", C.c_int64), ("n_entries", C.c_int64),
                ("cost", C.c_double), ("theta", C.c_double), ("solve_ms", C.c_double),
                ("total_d", C.c_int64), ("total_s", C.c_int64)]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def phase_cap(eps: float) -> int:
    """phase_bound + 8 (assignment.cpp:326, assignment.hpp:51)."""
    import math
    return int(math.ceil((1.0 + 2.0 * eps) / (eps * eps))) + 8


class Oracle:
    _inst = None

    @classmethod
    def get(cls) -> "Oracle":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        lib = C.CDLL(ORACLE_SO)
        self.lib = lib
        lib.orc_fnv1a64.restype = C.c_uint64
        lib.orc_fnv1a64.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        lib.orc_splitmix64.restype = C.c_uint64
        lib.orc_splitmix64.argtypes = [C.c_uint64]
        lib.orc_raw_stream.argtypes = [C.c_uint64, C.c_int64, _u64p]
        lib.orc_uniform_square_points.argtypes = [C.c_int32, C.c_uint64, _f64p, _f64p, _f64p, _f64p]
        lib.orc_gen_uniform_square.argtypes = [C.c_int32, C.c_uint64, _f64p]
        lib.orc_points_cost.restype = C.c_double
        lib.orc_points_cost.argtypes = [C.c_double] * 4
        lib.orc_scaled_floor.restype = C.c_int64
        lib.orc_scaled_floor.argtypes = [C.c_double, C.c_double]
        lib.orc_units.argtypes = [C.c_double, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.orc_scale_round_costs.argtypes = [C.c_int32, C.c_int32, _f64p, C.c_double, _i32p,
                                              C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.orc_mnist_sample.argtypes = [C.c_uint32, C.c_int32, C.c_uint64, _u32p]
        lib.orc_mnist_cost.argtypes = [C.c_int32, _u8p, _f64p]
        lib.orc_gen_random_ot_rational.argtypes = [C.c_int32, C.c_int32, C.c_uint64, _i64p, _i64p, _f64p]
        sol = [C.c_int32, C.c_int32]
        outs = [C.c_double, _i32p, _i32p, _i64p, _i64p, _i64p, C.c_int64, C.POINTER(_OrcStats)]
        lib.orc_solve_assignment.argtypes = sol + [_f64p] + outs
        lib.orc_solve_rounded.argtypes = sol + [_i32p] + outs
        lib.orc_matching_cost.restype = C.c_double
        lib.orc_matching_cost.argtypes = [C.c_int32, C.c_int32, _f64p, _i32p]

    # -- instances --
    def uniform_square_points(self, n: int, seed: int):
        ax, ay, bx, by = (np.empty(n, np.float64) for _ in range(4))
        st = self.lib.orc_uniform_square_points(n, seed, ax, ay, bx, by)
        if st:
            raise OracleError(st)
        return ax, ay, bx, by

    def gen_uniform_square(self, n: int, seed: int) -> np.ndarray:
        cost = np.empty((n, n), np.float64)
        st = self.lib.orc_gen_uniform_square(n, seed, cost)
        if st:
            raise OracleError(st)
        return cost

    def raw_stream(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        self.lib.orc_raw_stream(seed, count, out)
        return out

    def mnist_sample(self, count: int, n: int, seed: int) -> np.ndarray:
        out = np.empty(2 * n, np.uint32)
        st = self.lib.orc_mnist_sample(count, n, seed, out)
        if st:
            raise OracleError(st)
        return out

    def mnist_cost(self, images_2n: np.ndarray) -> np.ndarray:
        n = images_2n.shape[0] // 2
        cost = np.empty((n, n), np.float64)
        st = self.lib.orc_mnist_cost(n, np.ascontiguousarray(images_2n, np.uint8), cost)
        if st:
            raise OracleError(st)
        return cost

    def random_ot_rational(self, n_a: int, n_b: int, seed: int):
        wa, wb = np.empty(n_a, np.int64), np.empty(n_b, np.int64)
        cost = np.empty((n_a, n_b), np.float64)
        st = self.lib.orc_gen_random_ot_rational(n_a, n_b, seed, wa, wb, cost)
        if st:
            raise OracleError(st)
        return wa, wb, cost

    # -- rounding --
    def scaled_floor(self, c: float, eps: float) -> int:
        return int(self.lib.orc_scaled_floor(c, eps))

    def units(self, eps: float):
        uf, uc = C.c_int32(), C.c_int32()
        st = self.lib.orc_units(eps, C.byref(uf), C.byref(uc))
        if st:
            raise OracleError(st)
        return uf.value, uc.value

    def scale_round_costs(self, cost: np.ndarray, eps: float):
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        k = np.empty((n_a, n_b), np.int32)
        uf, uc = C.c_int32(), C.c_int32()
        st = self.lib.orc_scale_round_costs(n_a, n_b, cost, eps, k, C.byref(uf), C.byref(uc))
        if st:
            raise OracleError(st)
        return k, uf.value, uc.value

    # -- solver --
    def _outs(self, n_a, n_b, eps):
        ia, ib = max(n_a, n_b), min(n_a, n_b)
        cap = min(phase_cap(eps) + 1, 1 << 22)  # free_counts kept for the first 4M phases
        return (np.empty(n_a, np.int32), np.empty(n_b, np.int32), np.empty(ia, np.int64),
                np.empty(ib, np.int64), np.zeros(cap, np.int64), cap)

    def solve_assignment(self, cost: np.ndarray, eps: float) -> AssignResult:
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        ma, mb, ya, yb, fc, cap = self._outs(n_a, n_b, eps)
        s = _OrcStats()
        st = self.lib.orc_solve_assignment(n_a, n_b, cost, eps, ma, mb, ya, yb, fc, cap, C.byref(s))
        if st:
            raise OracleError(st)
        return AssignResult(ma, mb, ya, yb, fc[: s.phases].copy(), s.phases, s.sum_ni,
                            bool(s.swapped), bool(s.full_match_termination), s.cost)

    def solve_rounded(self, kT: np.ndarray, eps: float) -> AssignResult:
        """Solve on a B-major int32 k^T (n_b x n_a, n_b <= n_a)."""
        kT = np.ascontiguousarray(kT, np.int32)
        n_b, n_a = kT.shape
        ma, mb, ya, yb, fc, cap = self._outs(n_a, n_b, eps)
        s = _OrcStats()
        st = self.lib.orc_solve_rounded(n_a, n_b, kT, eps, ma, mb, ya, yb, fc, cap, C.byref(s))
        if st:
            raise OracleError(st)
        return AssignResult(ma, mb, ya, yb, fc[: s.phases].copy(), s.phases, s.sum_ni,
                            bool(s.swapped), bool(s.full_match_termination), 0.0)

    def matching_cost(self, cost: np.ndarray, match_of_a: np.ndarray) -> float:
        cost = np.ascontiguousarray(cost, np.float64)
        return float(self.lib.orc_matching_cost(cost.shape[0], cost.shape[1], cost,
                                                np.ascontiguousarray(match_of_a, np.int32)))


class Reference:
    """The unmodified reference library (oracle/_ref/libotpr_ref.so)."""
    _inst = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def get(cls) -> "Reference":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        lib = C.CDLL(REF_SO)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_gen_uniform_square.argtypes = [C.c_int32, C.c_uint64, _f64p]
        lib.ref_scale_round_costs.argtypes = [C.c_int32, C.c_int32, _f64p, C.c_double, _i32p,
                                              C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.ref_scaled_floor.restype = C.c_int64
        lib.ref_scaled_floor.argtypes = [C.c_double, C.c_double]
        outs = [_i32p, _i32p, _i64p, _i64p, _i64p, C.c_int64, C.POINTER(_RefStats)]
        lib.ref_solve_assignment.argtypes = [C.c_int32, C.c_int32, _f64p, C.c_double, C.c_int] + outs
        lib.ref_solve_uniform_square.argtypes = [C.c_int32, C.c_uint64, C.c_double, C.c_int, C.c_int] + outs
        lib.ref_solve_assignment_groups.argtypes = ([C.c_int32, C.c_int32, _f64p, C.c_double, _i32p, _i32p,
                                                     C.c_int32] + outs)
        lib.ref_load_mnist_pair.argtypes = [C.c_char_p, C.c_int32, C.c_uint64, _f64p]
        lib.ref_solve_mnist.argtypes = ([C.c_char_p, C.c_int32, C.c_uint64, C.c_double, C.c_int] + outs
                                        + [C.POINTER(C.c_double)])
        lib.ref_solve_ot_rational.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_double, _i32p, _i32p,
                                              _f64p, C.c_int64, _i64p, C.c_int64, C.POINTER(_RefOtStats)]
        lib.ref_gen_random_ot_rational.argtypes = [C.c_int32, C.c_int32, C.c_uint64, _f64p, _f64p, _f64p]
        lib.ref_solve_ot.argtypes = [C.c_int32, C.c_int32, _f64p, _f64p, _f64p, C.c_double, _i32p, _i32p,
                                     _f64p, C.c_int64, _i64p, C.c_int64, C.POINTER(_RefOtStats)]
        lib.ref_scale_and_round.argtypes = [C.c_int32, C.c_int32, _f64p, _f64p, _f64p, C.c_double, _i64p,
                                            _i64p, C.POINTER(C.c_double)]
        flat = [_i32p, _i64p, _i64p, _i64p, _i32p, _i64p, _i32p, _i64p, _i64p, _i64p]
        lib.ref_solve_copy_matching.argtypes = ([C.c_int32, C.c_int32, _i32p, C.c_double, C.c_int32,
                                                 C.c_int32, _i64p, _i64p, C.c_double, C.c_int32, _i64p,
                                                 _i64p, C.c_int64, _i64p, C.c_int64, _i64p, _i64p]
                                                + flat + [C.c_int64, _i64p])
        lib.ref_check_cluster.argtypes = ([C.c_int32, C.c_int32, _i32p, C.c_int32, _i64p, _i64p] + flat
                                          + [C.c_int32, C.POINTER(C.c_int64), C.c_char_p, C.c_int32])

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def gen_uniform_square(self, n: int, seed: int) -> np.ndarray:
        cost = np.empty((n, n), np.float64)
        self._check(self.lib.ref_gen_uniform_square(n, seed, cost))
        return cost

    def scaled_floor(self, c: float, eps: float) -> int:
        return int(self.lib.ref_scaled_floor(c, eps))

    def scale_round_costs(self, cost: np.ndarray, eps: float):
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        k = np.empty((n_a, n_b), np.int32)
        uf, uc = C.c_int32(), C.c_int32()
        self._check(self.lib.ref_scale_round_costs(n_a, n_b, cost, eps, k, C.byref(uf), C.byref(uc)))
        return k, uf.value, uc.value

    def _outs(self, n_a, n_b, eps):
        ia, ib = max(n_a, n_b), min(n_a, n_b)
        cap = min(phase_cap(eps) + 1, 1 << 22)  # free_counts kept for the first 4M phases
        return (np.empty(n_a, np.int32), np.empty(n_b, np.int32), np.empty(ia, np.int64),
                np.empty(ib, np.int64), np.zeros(cap, np.int64), cap)

    def _result(self, ma, mb, ya, yb, fc, s) -> AssignResult:
        return AssignResult(ma, mb, ya, yb, fc[: s.phases].copy(), s.phases, s.sum_ni,
                            bool(s.swapped), bool(s.full_match_termination), s.cost,
                            s.solve_ms, s.round_ms)

    def solve_assignment(self, cost: np.ndarray, eps: float, threads: int = 1) -> AssignResult:
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        ma, mb, ya, yb, fc, cap = self._outs(n_a, n_b, eps)
        s = _RefStats()
        self._check(self.lib.ref_solve_assignment(n_a, n_b, cost, eps, threads, ma, mb, ya, yb, fc, cap,
                                                  C.byref(s)))
        return self._result(ma, mb, ya, yb, fc, s)

    def solve_assignment_groups(self, cost: np.ndarray, eps: float, demand_groups, supply_groups,
                                check_invariants: bool = False) -> AssignResult:
        """Copy mode (assignment.cpp:81-103, :241-250), threads = 1."""
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        ma, mb, ya, yb, fc, cap = self._outs(n_a, n_b, eps)
        s = _RefStats()
        dg = np.ascontiguousarray(demand_groups, np.int32)
        sg = np.ascontiguousarray(supply_groups, np.int32)
        self._check(self.lib.ref_solve_assignment_groups(n_a, n_b, cost, eps, dg, sg, int(check_invariants),
                                                         ma, mb, ya, yb, fc, cap, C.byref(s)))
        return self._result(ma, mb, ya, yb, fc, s)

    def solve_uniform_square(self, n: int, seed: int, eps: float, threads: int = 1,
                             time_rounding: bool = False) -> AssignResult:
        ma, mb, ya, yb, fc, cap = self._outs(n, n, eps)
        s = _RefStats()
        self._check(self.lib.ref_solve_uniform_square(n, seed, eps, threads, int(time_rounding), ma, mb, ya,
                                                      yb, fc, cap, C.byref(s)))
        return self._result(ma, mb, ya, yb, fc, s)

    def load_mnist_pair(self, path: str, n: int, seed: int) -> np.ndarray:
        cost = np.empty((n, n), np.float64)
        self._check(self.lib.ref_load_mnist_pair(path.encode(), n, seed, cost))
        return cost

    def solve_mnist(self, path: str, n: int, seed: int, eps: float, threads: int = 1) -> AssignResult:
        ma, mb, ya, yb, fc, cap = self._outs(n, n, eps)
        s = _RefStats()
        load_ms = C.c_double()
        self._check(self.lib.ref_solve_mnist(path.encode(), n, seed, eps, threads, ma, mb, ya, yb, fc, cap,
                                             C.byref(s), C.byref(load_ms)))
        r = self._result(ma, mb, ya, yb, fc, s)
        r.extra["load_ms"] = load_ms.value
        return r

    def gen_random_ot_rational(self, n_a: int, n_b: int, seed: int):
        mu, nu = np.empty(n_a), np.empty(n_b)
        cost = np.empty((n_a, n_b))
        self._check(self.lib.ref_gen_random_ot_rational(n_a, n_b, seed, mu, nu, cost))
        return mu, nu, cost

    def solve_ot(self, mu, nu, cost, eps: float, entry_cap: int | None = None):
        """otpr::solve_ot on the given instance (masses as given, no renormalisation)."""
        mu = np.ascontiguousarray(mu, np.float64)
        nu = np.ascontiguousarray(nu, np.float64)
        cost = np.ascontiguousarray(cost, np.float64)
        n_a, n_b = cost.shape
        cap_e = entry_cap or (n_a + n_b) * 4 + 16
        ea, eb, em = np.empty(cap_e, np.int32), np.empty(cap_e, np.int32), np.empty(cap_e)
        fcap = min(phase_cap(eps / 3.0) + 1, 1 << 22)
        fc = np.zeros(fcap, np.int64)
        s = _RefOtStats()
        self._check(self.lib.ref_solve_ot(n_a, n_b, mu, nu, cost, eps, ea, eb, em, cap_e, fc, fcap,
                                          C.byref(s)))
        ne = min(s.n_entries, cap_e)
        return {"phases": s.phases, "sum_ni": s.sum_ni, "cost": s.cost, "theta": s.theta,
                "solve_ms": s.solve_ms, "n_entries": s.n_entries, "total_d": s.total_d,
                "total_s": s.total_s, "a": ea[:ne].copy(), "b": eb[:ne].copy(), "mass": em[:ne].copy(),
                "free_counts": fc[: s.phases].copy()}

    def scale_and_round(self, mu, nu, cost, eps: float):
        mu = np.ascontiguousarray(mu, np.float64)
        nu = np.ascontiguousarray(nu, np.float64)
        cost = np.ascontiguousarray(cost, np.float64)
        d, s = np.empty(len(mu), np.int64), np.empty(len(nu), np.int64)
        th = C.c_double()
        self._check(self.lib.ref_scale_and_round(len(mu), len(nu), mu, nu, cost, eps, d, s, C.byref(th)))
        return d, s, th.value

    def solve_ot_rational(self, n_a: int, n_b: int, seed: int, eps: float, entry_cap: int | None = None):
        cap_e = entry_cap or (n_a + n_b) * 4
        ea, eb, em = np.empty(cap_e, np.int32), np.empty(cap_e, np.int32), np.empty(cap_e)
        fcap = min(phase_cap(eps / 3.0) + 1, 1 << 22)
        fc = np.zeros(fcap, np.int64)
        s = _RefOtStats()
        self._check(self.lib.ref_solve_ot_rational(n_a, n_b, seed, eps, ea, eb, em, cap_e, fc, fcap,
                                                   C.byref(s)))
        ne = min(s.n_entries, cap_e)
        return {"phases": s.phases, "sum_ni": s.sum_ni, "cost": s.cost, "theta": s.theta,
                "solve_ms": s.solve_ms, "n_entries": s.n_entries, "total_d": s.total_d,
                "total_s": s.total_s, "a": ea[:ne].copy(), "b": eb[:ne].copy(), "mass": em[:ne].copy(),
                "free_counts": fc[: s.phases].copy()}


# ---- copy/cluster solver of the reference (ot.hpp:52-151) -------------------
FLAT_KEYS = ("dem_off", "dem_y", "dem_free", "flow_off", "flow_b", "flow_cnt", "sup_off", "sup_y",
             "sup_free", "sup_matched")


def _ref_copy_matching(self, k, ceps, uf, uc, d, s, eps, check=True, phase_cap=4096):
    """otpr::solve_copy_matching on CopyInstance{k, d, s}: final flow,
    free_counts, stats, the per-phase flow matrices (observer) and the final
    ClusterState in the flat layout of include/otprg.h."""
    k = np.ascontiguousarray(k, np.int32)
    d = np.ascontiguousarray(d, np.int64)
    s = np.ascontiguousarray(s, np.int64)
    n_a, n_b = k.shape
    flow = np.zeros((n_a, n_b), np.int64)
    fc = np.zeros(1 << 16, np.int64)
    pf = np.zeros((phase_cap, n_a, n_b), np.int64)
    pni = np.zeros(phase_cap, np.int64)
    st3 = np.zeros(3, np.int64)
    cap = int(d.sum() + s.sum()) * 2 + 4 * (n_a + n_b) + 16
    fl = dict(dem_off=np.zeros(n_a + 1, np.int32), dem_y=np.zeros(cap, np.int64),
              dem_free=np.zeros(cap, np.int64), flow_off=np.zeros(cap + 1, np.int64),
              flow_b=np.zeros(cap, np.int32), flow_cnt=np.zeros(cap, np.int64),
              sup_off=np.zeros(n_b + 1, np.int32), sup_y=np.zeros(cap, np.int64),
              sup_free=np.zeros(cap, np.int64), sup_matched=np.zeros(cap, np.int64))
    sizes = np.zeros(3, np.int64)
    self._check(self.lib.ref_solve_copy_matching(n_a, n_b, k, ceps, uf, uc, d, s, eps, int(check), flow,
                                                 fc, len(fc), pf, phase_cap, pni, st3,
                                                 *[fl[x] for x in FLAT_KEYS], cap, sizes))
    nd, nf, ns = (int(x) for x in sizes)
    assert max(nd, nf, ns) <= cap
    state = dict(dem_off=fl["dem_off"], dem_y=fl["dem_y"][:nd], dem_free=fl["dem_free"][:nd],
                 flow_off=fl["flow_off"][: nd + 1], flow_b=fl["flow_b"][:nf], flow_cnt=fl["flow_cnt"][:nf],
                 sup_off=fl["sup_off"], sup_y=fl["sup_y"][:ns], sup_free=fl["sup_free"][:ns],
                 sup_matched=fl["sup_matched"][:ns])
    ph = int(st3[0])
    return dict(flow=flow, free_counts=fc[:ph].copy(), phases=ph, sum_ni=int(st3[1]),
                full_match_termination=bool(st3[2]), phase_flows=pf[: min(ph, phase_cap)].copy(),
                phase_ni=pni[: min(ph, phase_cap)].copy(), state=state)


def _ref_check_cluster(self, k, uc, d, s, state: dict, which: int):
    """otpr::check_cluster_invariant (0) / check_cluster_feasibility (1)."""
    k = np.ascontiguousarray(k, np.int32)
    n_a, n_b = k.shape
    cnt = C.c_int64()
    buf = C.create_string_buffer(1 << 16)
    arrs = [np.ascontiguousarray(state[x], np.int32 if x in ("dem_off", "flow_b", "sup_off") else np.int64)
            for x in FLAT_KEYS]
    self._check(self.lib.ref_check_cluster(n_a, n_b, k, uc, np.ascontiguousarray(d, np.int64),
                                           np.ascontiguousarray(s, np.int64), *arrs, which, C.byref(cnt),
                                           buf, len(buf)))
    msgs = buf.value.decode().split("\n") if cnt.value else []
    return msgs[: cnt.value]


Reference.solve_copy_matching = _ref_copy_matching
Reference.check_cluster = _ref_check_cluster
