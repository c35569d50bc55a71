"""Host-side mirror of the reference's assignment API (namespace ``otpr``).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/otpr/{core,assignment,errors,instances}.hpp, so
code (and tests) written against the reference read the same here:

    inst = gen_uniform_square(10_000, seed=1)
    matching, stats = solve_assignment(inst, AssignmentOptions(eps=0.01))

Every solve runs on the GPU through the C ABI (include/otprg.h ->
paper_2203_03732_b200/lib/libotprg.so).  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N

K_UNMATCHED = -1


# ---- errors (include/otpr/errors.hpp:9-37) -------------------------------
class ParameterError(ValueError):
    """Out-of-range or inconsistent caller-supplied parameters."""


class InputError(RuntimeError):
    """Malformed or unusable input data."""


class FormatError(InputError):
    """Byte-level file format problems."""


class NumericalError(RuntimeError):
    """Numerical failure of an iterative method."""


class InvariantViolation(RuntimeError):
    """A solver state check failed (a bug, not bad input)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure (no reference counterpart)."""


_STATUS_EXC = {N.PARAMETER: ParameterError, N.INPUT: InputError, N.NUMERICAL: NumericalError,
               N.INVARIANT: InvariantViolation, N.DEVICE: DeviceError,
               N.ABORTED: DeviceError}  # (an observer's own exception is re-raised instead)


# ---- data model (include/otpr/core.hpp) ----------------------------------
@dataclass
class AssignmentInstance:
    """core.hpp:69-81.  Either a dense row-major cost (rows = A, cols = B) or,
    as a B200-native extension, 2-D point sets whose cost is
    gen_uniform_square's Euclidean/sqrt(2) (instances.cpp:70-75), evaluated
    on the device without materialising n_a x n_b doubles."""
    n_a: int
    n_b: int
    cost: Optional[np.ndarray] = None      # (n_a, n_b) float64
    pts_a: Optional[np.ndarray] = None     # (n_a, 2) float64
    pts_b: Optional[np.ndarray] = None     # (n_b, 2) float64
    norm_factor: float = 1.0
    seed: int = 0
    img_a: Optional[np.ndarray] = None     # (n_a, dim) uint8: L1/2 cost of normalised images
    img_b: Optional[np.ndarray] = None     # (n_b, dim) uint8   (load_mnist_pair, instances.cpp:80-144)

    def validate(self) -> None:
        """core.cpp:10-24."""
        if self.n_a < 1 or self.n_b < 1:
            raise ParameterError("instance needs at least one vertex per side")
        if self.cost is not None:
            if self.cost.shape != (self.n_a, self.n_b):
                raise ParameterError("cost matrix dimensions do not match n_a x n_b")
            bad = ~((self.cost >= 0.0) & (self.cost <= 1.0))
            if bad.any():
                a, b = np.argwhere(bad)[0]
                raise ParameterError(f"cost entry outside [0,1] at ({a},{b}): {self.cost[a, b]:f}")
        elif (self.pts_a is None or self.pts_b is None) and (self.img_a is None or self.img_b is None):
            raise ParameterError("instance has neither a cost matrix, point sets nor images")

    def dense_cost(self) -> np.ndarray:
        if self.cost is not None:
            return self.cost
        if self.img_a is not None:
            return l1_cost(self.img_a, self.img_b)
        return points_cost(self.pts_a, self.pts_b)


@dataclass
class ScaledCosts:
    """core.hpp:85-96."""
    eps: float
    k: np.ndarray  # (n_a, n_b) int32
    unit_floor: int
    unit_ceil: int

    def dual_bound(self) -> int:
        return int(self.unit_ceil) + 2


@dataclass
class DualState:
    """core.hpp:109-114 (integer eps-units)."""
    y_a: np.ndarray
    y_b: np.ndarray

    def sum_abs(self) -> int:
        return int(np.abs(self.y_a).sum() + np.abs(self.y_b).sum())


@dataclass
class Matching:
    """core.hpp:117-138."""
    match_of_a: np.ndarray
    match_of_b: np.ndarray

    @classmethod
    def empty(cls, n_a: int, n_b: int) -> "Matching":
        return cls(np.full(n_a, K_UNMATCHED, np.int32), np.full(n_b, K_UNMATCHED, np.int32))

    def has_a(self, a: int) -> bool:
        return self.match_of_a[a] != K_UNMATCHED

    def has_b(self, b: int) -> bool:
        return self.match_of_b[b] != K_UNMATCHED

    def link(self, a: int, b: int) -> None:
        self.match_of_a[a] = b
        self.match_of_b[b] = a

    def size(self) -> int:
        return int((self.match_of_a != K_UNMATCHED).sum())

    def validate(self) -> None:
        """core.cpp:77-93."""
        n_a, n_b = len(self.match_of_a), len(self.match_of_b)
        for a, b in enumerate(self.match_of_a):
            if b == K_UNMATCHED:
                continue
            if b < 0 or b >= n_b or self.match_of_b[b] != a:
                raise InvariantViolation(f"matching is not mutually consistent at a={a}")
        for b, a in enumerate(self.match_of_b):
            if a == K_UNMATCHED:
                continue
            if a < 0 or a >= n_a or self.match_of_a[a] != b:
                raise InvariantViolation(f"matching is not mutually consistent at b={b}")


@dataclass
class SolveStats:
    """assignment.hpp:35-53, plus device measurements."""
    phases: int = 0
    free_counts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    sum_ni: int = 0
    duals_final: Optional[DualState] = None
    swapped: bool = False
    full_match_termination: bool = False
    device: dict = field(default_factory=dict)

    @staticmethod
    def phase_bound(eps: float) -> int:
        return int(math.ceil((1.0 + 2.0 * eps) / (eps * eps)))

    @staticmethod
    def sum_ni_bound(eps: float, n: int) -> int:
        return int(math.ceil(float(n) * (1.0 + 2.0 * eps) / eps))


@dataclass
class PhaseWorkset:
    """assignment.hpp:20-33 (internal orientation): B', E' (admissible a of
    every free b, ascending), A', and the phase products M', A'', M''."""
    b_free: np.ndarray
    e_admissible: list
    a_touched: np.ndarray
    m_prime: list
    a_double: list
    m_double: list

    def edge_count(self) -> int:
        return int(sum(len(e) for e in self.e_admissible))


@dataclass
class PhaseSnapshot:
    """assignment.hpp:57-67: handed to the observer after each phase, in the
    solver's internal orientation."""
    phase: int
    costs: "ScaledCosts"
    duals: DualState
    matching: Matching
    workset: PhaseWorkset
    sum_abs_before: int
    sum_abs_after: int


@dataclass
class FeasibilityReport:
    """assignment.hpp:116-120.  The device suite reports the first violation
    in the reference's order (the message check_invariants throws) and the
    number of violations; ``violations`` holds that first message, ``count``
    the total."""
    violations: list = field(default_factory=list)
    notes: list = field(default_factory=list)
    count: int = 0
    kind: int = 0
    a: int = -1
    b: int = -1

    def ok(self) -> bool:
        return not self.violations


_VIOL_MSG = {
    1: "matching is not mutually consistent at a={a}",
    2: "matching is not mutually consistent at b={b}",
    3: "demand dual positive at a={a}",
    4: "free demand vertex with nonzero dual at a={a}",
    5: "demand dual magnitude exceeds bound at a={a}",
    6: "supply dual negative at b={b}",
    7: "supply dual magnitude exceeds bound at b={b}",
    8: "matching edge not tight at ({a},{b}): Y(a)+Y(b)={s} k={k}",
    9: "dual sum exceeds rounded cost allowance at ({a},{b}): Y(a)+Y(b)={s} k={k}",
}


def _report(f: "N.Feasibility") -> FeasibilityReport:
    """verify_feasibility's report strings (assignment.cpp:270-311, core.cpp:69-86)."""
    if f.violations == 0:
        return FeasibilityReport()
    msg = _VIOL_MSG[f.kind].format(a=f.a, b=f.b, s=f.sum, k=f.k)
    return FeasibilityReport(violations=[msg], count=int(f.violations), kind=int(f.kind), a=int(f.a),
                             b=int(f.b))


@dataclass
class AssignmentOptions:
    """assignment.hpp:69-90.  ``threads`` is accepted and ignored: the device
    path always has threads=1 (deterministic) semantics.  ``observer`` and
    ``check_invariants`` switch to the host-synced stepping loop (one phase
    per launch; the device invariant suite after every phase; the
    PhaseSnapshot built from device exports), as the reference runs them
    inside solve_oriented (assignment.cpp:344-355).  ``storage`` selects the device width of the rounded matrix.
    ``costs`` (2-D point instances): "matrix" materialises the rounded kT in HBM, "on_the_fly" never
    does (the scans round the point costs through the exact threshold table; the
    sharded driver with one shard), "auto" picks the matrix when it fits in free HBM."""
    eps: float = 0.1
    threads: int = 1
    check_invariants: bool = False
    observer: Optional[Callable] = None
    demand_groups: Optional[np.ndarray] = None
    supply_groups: Optional[np.ndarray] = None
    storage: str = "auto"
    device: int = 0
    costs: str = "auto"


# ---- device context ------------------------------------------------------
class Solver:
    """Owns one otprg_ctx (device buffers reused across solves)."""

    def __init__(self, device: int = 0):
        self._L = N.lib()
        self._ctx = C.c_void_p()
        st = self._L.otprg_create(device, C.byref(self._ctx))
        if st:
            raise DeviceError(f"otprg_create(device={device}) failed with status {st}")
        self.device = device
        self._keep = ()

    def close(self) -> None:
        if self._ctx:
            self._L.otprg_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, st: int):
        msg = self._L.otprg_last_error(self._ctx).decode()
        raise _STATUS_EXC.get(st, DeviceError)(msg)

    def _problem(self, inst: AssignmentInstance, eps: float, storage: str) -> N.Problem:
        p = N.Problem()
        p.n_a, p.n_b, p.eps = inst.n_a, inst.n_b, float(eps)
        if storage not in N.STORAGE:
            raise ParameterError(f"unknown storage {storage!r}")
        p.storage = N.STORAGE[storage]
        if inst.cost is not None:
            cost = np.ascontiguousarray(inst.cost, np.float64)
            if cost.shape != (inst.n_a, inst.n_b):
                raise ParameterError("cost matrix dimensions do not match n_a x n_b")
            p.cost_kind = N.COST_DENSE_F64
            p.cost = cost.ctypes.data
            self._keep = (cost,)
        elif inst.img_a is not None and inst.img_b is not None:
            ia = np.ascontiguousarray(inst.img_a, np.uint8).reshape(inst.n_a, -1)
            ib = np.ascontiguousarray(inst.img_b, np.uint8).reshape(inst.n_b, -1)
            if ia.shape[1] != ib.shape[1]:
                raise ParameterError("image dimensions differ between the sides")
            p.cost_kind = N.COST_L1_U8
            p.img_a, p.img_b, p.dim = ia.ctypes.data, ib.ctypes.data, ia.shape[1]
            self._keep = (ia, ib)
        elif inst.pts_a is not None and inst.pts_b is not None:
            pa = np.ascontiguousarray(inst.pts_a, np.float64).reshape(inst.n_a, 2)
            pb = np.ascontiguousarray(inst.pts_b, np.float64).reshape(inst.n_b, 2)
            p.cost_kind = N.COST_POINTS2D
            p.pts_a, p.pts_b = pa.ctypes.data, pb.ctypes.data
            self._keep = (pa, pb)
        else:
            raise ParameterError("instance has neither a cost matrix nor point sets")
        return p

    def _result(self, n_a: int, n_b: int, eps: float):
        ia, ib = max(n_a, n_b), min(n_a, n_b)
        cap = min(SolveStats.phase_bound(eps) + 10, N.MAX_PHASES + 2)
        bufs = dict(match_of_a=np.empty(n_a, np.int32), match_of_b=np.empty(n_b, np.int32),
                    y_a=np.empty(ia, np.int64), y_b=np.empty(ib, np.int64),
                    free_counts=np.zeros(cap, np.int64))
        r = N.Result()
        for k, v in bufs.items():
            setattr(r, k, v.ctypes.data)
        r.free_cap = cap
        return r, bufs

    def prepare(self, inst: AssignmentInstance, eps: float, storage: str = "auto") -> dict:
        p = self._problem(inst, eps, storage)
        r = N.Result()
        st = self._L.otprg_prepare(self._ctx, C.byref(p), C.byref(r))
        if st:
            self._raise(st)
        self._prepared = (inst.n_a, inst.n_b, eps)
        return {"build_ms": r.build_ms, "width": r.width}

    def solve_prepared(self):
        n_a, n_b, eps = self._prepared
        r, bufs = self._result(n_a, n_b, eps)
        st = self._L.otprg_solve_prepared(self._ctx, C.byref(r))
        if st:
            self._raise(st)
        return self._pack(r, bufs)

    # -- stepping (host-synced) form --
    def begin(self) -> None:
        st = self._L.otprg_begin(self._ctx)
        if st:
            self._raise(st)

    def step(self, max_phases: int) -> tuple[int, bool]:
        """Run until ``max_phases`` phases executed in total (<=0: to the end)."""
        done, fin = C.c_int64(), C.c_int32()
        st = self._L.otprg_step(self._ctx, max_phases, C.byref(done), C.byref(fin))
        if st:
            self._raise(st)
        return int(done.value), bool(fin.value)

    def snapshot(self):
        n_a, n_b, eps = self._prepared
        r, bufs = self._result(n_a, n_b, eps)
        st = self._L.otprg_snapshot(self._ctx, C.byref(r))
        if st:
            self._raise(st)
        return self._pack(r, bufs)

    def finish(self):
        n_a, n_b, eps = self._prepared
        r, bufs = self._result(n_a, n_b, eps)
        st = self._L.otprg_finish(self._ctx, C.byref(r))
        if st:
            self._raise(st)
        return self._pack(r, bufs)

    def solve(self, inst: AssignmentInstance, opt: AssignmentOptions):
        p = self._problem(inst, opt.eps, opt.storage)
        r, bufs = self._result(inst.n_a, inst.n_b, opt.eps)
        st = self._L.otprg_solve_assignment(self._ctx, C.byref(p), C.byref(r))
        if st:
            self._raise(st)
        return self._pack(r, bufs)

    @staticmethod
    def _pack(r: N.Result, bufs: dict):
        m = Matching(bufs["match_of_a"], bufs["match_of_b"])
        stats = SolveStats(
            phases=int(r.phases), free_counts=bufs["free_counts"][: r.phases].copy(),
            sum_ni=int(r.sum_ni), duals_final=DualState(bufs["y_a"], bufs["y_b"]),
            swapped=bool(r.swapped), full_match_termination=bool(r.full_match_termination),
            device=dict(cost=r.cost, build_ms=r.build_ms, solve_ms=r.solve_ms,
                        phase1_ms=r.phase1_ms, loop_ms=r.loop_ms, solve_d2h_ms=r.solve_d2h_ms,
                        bytes_touched=int(r.bytes_touched),
                        bytes_alg=int(r.bytes_alg), width=int(r.width),
                        chain_stats=dict(zip(
                            ("fresh", "takeover", "cache_hit", "cache_exhaust", "scan_past_cache",
                             "rescan", "rowmin_skip", "proposals"), list(r.chain_stats))),
                        gpu_launches=int(r.gpu_launches), refill_rounds=int(r.refill_rounds),
                        n_shards=int(r.n_shards)))
        return m, stats

    def scale_round_costs(self, inst: AssignmentInstance, eps: float, storage: str = "auto") -> ScaledCosts:
        p = self._problem(inst, eps, storage)
        k = np.empty((inst.n_a, inst.n_b), np.int32)
        uf, uc = C.c_int32(), C.c_int32()
        st = self._L.otprg_scale_round_costs(self._ctx, C.byref(p), k.ctypes.data, C.byref(uf),
                                             C.byref(uc))
        if st:
            self._raise(st)
        return ScaledCosts(eps, k, uf.value, uc.value)

    # -- invariant suite / workset export --
    def verify_feasibility(self) -> FeasibilityReport:
        """verify_feasibility on the device state between phases (internal
        orientation)."""
        f = N.Feasibility()
        st = self._L.otprg_verify_feasibility(self._ctx, C.byref(f))
        if st:
            self._raise(st)
        return _report(f)

    def verify_result(self, duals: DualState, m: Matching) -> FeasibilityReport:
        """verify_feasibility of a result state (internal orientation,
        pre-completion matching) against this solver's prepared rounded costs
        on the device (no host k matrix: the n = 100k check)."""
        ya = np.ascontiguousarray(duals.y_a, np.int64)
        yb = np.ascontiguousarray(duals.y_b, np.int64)
        ma = np.ascontiguousarray(m.match_of_a, np.int32)
        mb = np.ascontiguousarray(m.match_of_b, np.int32)
        f = N.Feasibility()
        st = self._L.otprg_verify_result(self._ctx, ya.ctypes.data, yb.ctypes.data, ma.ctypes.data,
                                         mb.ctypes.data, C.byref(f))
        if st:
            self._raise(st)
        return _report(f)

    def verify_host(self, sc: "ScaledCosts", duals: DualState, m: Matching) -> FeasibilityReport:
        k = np.ascontiguousarray(sc.k, np.int32)
        n_a, n_b = k.shape
        ya = np.ascontiguousarray(duals.y_a, np.int64)
        yb = np.ascontiguousarray(duals.y_b, np.int64)
        ma = np.ascontiguousarray(m.match_of_a, np.int32)
        mb = np.ascontiguousarray(m.match_of_b, np.int32)
        if len(ya) != n_a or len(yb) != n_b or len(ma) != n_a or len(mb) != n_b:
            raise ParameterError("state sizes do not match the cost matrix")
        f = N.Feasibility()
        st = self._L.otprg_verify_host(self._ctx, n_a, n_b, k.ctypes.data, int(sc.unit_ceil),
                                       ya.ctypes.data, yb.ctypes.data, ma.ctypes.data,
                                       mb.ctypes.data, C.byref(f))
        if st:
            self._raise(st)
        return _report(f)

    def admissible(self, n_b: int):
        """(B', E') of the current state: free b ascending and the admissible
        a of each, ascending (collect_workset, assignment.cpp:107-147)."""
        bfree = np.empty(n_b, np.int32)
        offs = np.empty(n_b + 1, np.int64)
        nf, ne = C.c_int64(), C.c_int64()
        st = self._L.otprg_admissible(self._ctx, bfree.ctypes.data, offs.ctypes.data, None, 0,
                                      C.byref(nf), C.byref(ne))
        if st:
            self._raise(st)
        alist = np.empty(max(int(ne.value), 1), np.int32)
        if ne.value:
            st = self._L.otprg_admissible(self._ctx, bfree.ctypes.data, offs.ctypes.data,
                                          alist.ctypes.data, alist.size, C.byref(nf), C.byref(ne))
            if st:
                self._raise(st)
        n = int(nf.value)
        return bfree[:n].copy(), [alist[offs[i]:offs[i + 1]].copy() for i in range(n)]

    def flush_l2(self) -> None:
        st = self._L.otprg_flush_l2(self._ctx)
        if st:
            self._raise(st)

    def set_trace(self, max_phases: int) -> None:
        st = self._L.otprg_set_trace(self._ctx, max_phases)
        if st:
            self._raise(st)

    def get_trace(self, phases: int) -> np.ndarray:
        """(phases, 16) uint64 device timeline; see include/otprg.h."""
        out = np.zeros((phases, 16), np.uint64)
        st = self._L.otprg_get_trace(self._ctx, out.ctypes.data, phases)
        if st:
            self._raise(st)
        return out

    def timer_start(self) -> None:
        st = self._L.otprg_timer_start(self._ctx)
        if st:
            self._raise(st)

    def timer_stop(self) -> float:
        ms = C.c_double()
        st = self._L.otprg_timer_stop(self._ctx, C.byref(ms))
        if st:
            self._raise(st)
        return float(ms.value)


_solvers: dict[int, Solver] = {}


def get_solver(device: int = 0) -> Solver:
    if device not in _solvers:
        _solvers[device] = Solver(device)
    return _solvers[device]


# ---- free functions mirroring the reference ------------------------------
def scaled_floor(c: float, eps: float) -> int:
    """core.cpp:26-32 (host)."""
    return int(N.lib().otprg_scaled_floor(c, eps))


def scale_round_costs(inst: AssignmentInstance, eps: float, storage: str = "auto",
                      device: int = 0) -> ScaledCosts:
    """core.cpp:34-53, computed on the device."""
    inst.validate()
    return get_solver(device).scale_round_costs(inst, eps, storage)


def _check_options(inst: AssignmentInstance, opt: AssignmentOptions) -> None:
    """assignment.cpp:370-383."""
    inst.validate()
    if not (opt.eps > 0.0 and opt.eps < 1.0):
        raise ParameterError("eps must lie in (0, 1)")
    if (opt.demand_groups is None) != (opt.supply_groups is None):
        raise ParameterError("copy mode needs both demand and supply groups")
    if opt.demand_groups is not None:
        if len(opt.demand_groups) != inst.n_a or len(opt.supply_groups) != inst.n_b:
            raise ParameterError("group map sizes do not match the instance")
        if inst.n_b > inst.n_a:
            raise ParameterError("copy mode requires n_b <= n_a")


def _matrix_fits(inst: AssignmentInstance, opt: AssignmentOptions) -> bool:
    """Whether the rounded matrix (uint16 rows padded to 256 entries, or
    uint32 for tiny eps) fits in the device's free memory with a 10 % margin."""
    ia, ib = max(inst.n_a, inst.n_b), min(inst.n_a, inst.n_b)
    width = 4 if opt.storage == "u32" or (0 < opt.eps < 1 and math.ceil(1.0 / opt.eps) + 2 > 65533) \
        else (1 if opt.storage == "u8" else 2)
    need = ib * ((ia + 511) // 512 * 512) * width
    free, total = C.c_uint64(), C.c_uint64()
    if N.lib().otprg_mem_info(opt.device, C.byref(free), C.byref(total)) != 0:
        raise DeviceError(f"cannot query the memory of device {opt.device}")
    return need <= 0.9 * free.value


def solve_assignment(inst: AssignmentInstance, opt: AssignmentOptions):
    """assignment.hpp:137-138 / assignment.cpp:368-400 -> (Matching, SolveStats)."""
    _check_options(inst, opt)
    if opt.costs not in ("auto", "matrix", "on_the_fly"):
        raise ParameterError(f"unknown costs mode {opt.costs!r}")
    if opt.observer is not None or opt.check_invariants or opt.demand_groups is not None:
        return _solve_debug(get_solver(opt.device), inst, opt)
    if inst.cost is None and (inst.pts_a is not None or inst.img_a is not None) and (
            opt.costs == "on_the_fly" or (opt.costs == "auto" and not _matrix_fits(inst, opt))):
        from .sharded import solve_assignment_sharded  # one shard, no kT anywhere
        return solve_assignment_sharded(inst, opt, 1, on_the_fly=True)
    return get_solver(opt.device).solve(inst, opt)


def _internal(m: Matching, swapped: bool) -> Matching:
    return Matching(m.match_of_b, m.match_of_a) if swapped else m


def _solve_debug(sv: Solver, inst: AssignmentInstance, opt: AssignmentOptions):
    """The host-synced form of solve_oriented (assignment.cpp:316-364): one
    device phase per step; after it the device invariant suite
    (check_invariants, :344-349) and the observer (:350-355) see the state in
    the internal orientation.  Results are those of the fused solve."""
    swapped = inst.n_b > inst.n_a
    n_b_int = min(inst.n_a, inst.n_b)
    grouped = opt.demand_groups is not None
    costs = None
    if opt.observer is not None:  # ScaledCosts in the internal orientation (prepares too)
        sc = sv.scale_round_costs(inst, opt.eps, opt.storage)
        costs = ScaledCosts(sc.eps, np.ascontiguousarray(sc.k.T) if swapped else sc.k,
                            sc.unit_floor, sc.unit_ceil)
    elif not grouped:
        sv.prepare(inst, opt.eps, opt.storage)
    sv._prepared = (inst.n_a, inst.n_b, opt.eps)
    if grouped:  # copy mode: its own phase step (assignment.cpp:81-103, :241-250)
        dg = np.ascontiguousarray(opt.demand_groups, np.int32)
        sg = np.ascontiguousarray(opt.supply_groups, np.int32)
        p = sv._problem(inst, opt.eps, opt.storage)
        st = sv._L.otprg_groups_begin(sv._ctx, C.byref(p), dg.ctypes.data, sg.ctypes.data)
        if st:
            sv._raise(st)
    else:
        sv.begin()
    threshold = opt.eps * float(min(inst.n_a, inst.n_b))
    m0, s0 = sv.snapshot()
    cur_m, cur_d = _internal(m0, swapped), s0.duals_final
    phase = 0
    while True:
        if opt.observer is not None:
            b_free, e_adm = sv.admissible(n_b_int)
        else:
            b_free = np.flatnonzero(cur_m.match_of_b == K_UNMATCHED).astype(np.int32)
            e_adm = None
        if float(len(b_free)) <= threshold:
            break
        if grouped and e_adm is not None:  # scan_grouped order (assignment.cpp:81-103)
            ma = cur_m.match_of_a
            part = np.where(ma >= 0, sg[np.maximum(ma, 0)], 0)
            order = np.lexsort((np.arange(len(dg)), part, (ma >= 0).astype(np.int64), dg))
            rank = np.empty(len(dg), np.int64)
            rank[order] = np.arange(len(dg))
            e_adm = [e[np.argsort(rank[e], kind="stable")] for e in e_adm]
        before = int(np.abs(cur_d.y_a).sum() + np.abs(cur_d.y_b).sum())
        if grouped:
            d64, f32 = C.c_int64(), C.c_int32()
            st = sv._L.otprg_groups_step(sv._ctx, C.byref(d64), C.byref(f32))
            if st:
                sv._raise(st)
            done = int(d64.value)
        else:
            done, _ = sv.step(phase + 1)
        if done != phase + 1:
            raise InvariantViolation(f"device loop stopped at phase {done}, expected {phase + 1}")
        phase = done
        prev_m = cur_m
        m1, s1 = sv.snapshot()
        cur_m, cur_d = _internal(m1, swapped), s1.duals_final
        if opt.check_invariants:
            rep = sv.verify_feasibility()
            if not rep.ok():
                raise InvariantViolation(f"phase {phase}: {rep.violations[0]}")
        if opt.observer is not None:
            m_prime, a_double, m_double = [], [], []
            for b in b_free:  # M' in B' order (the sequential greedy's order)
                a = int(cur_m.match_of_b[b])
                if a == K_UNMATCHED:
                    continue
                m_prime.append((a, int(b)))
                old_b = int(prev_m.match_of_a[a])
                if old_b != K_UNMATCHED:
                    a_double.append(a)
                    m_double.append((a, old_b))
            touched = np.unique(np.concatenate(e_adm)) if e_adm else np.zeros(0, np.int32)
            ws = PhaseWorkset(b_free, e_adm, touched.astype(np.int32), m_prime, a_double, m_double)
            after = int(np.abs(cur_d.y_a).sum() + np.abs(cur_d.y_b).sum())
            opt.observer(PhaseSnapshot(phase, costs, cur_d, cur_m, ws, before, after))
    if grouped:
        n_a, n_b, eps = sv._prepared
        r, bufs = sv._result(n_a, n_b, eps)
        st = sv._L.otprg_groups_finish(sv._ctx, C.byref(r))
        if st:
            sv._raise(st)
        return Solver._pack(r, bufs)
    return sv.finish()


def verify_feasibility(sc: "ScaledCosts", duals: DualState, m: Matching,
                       device: int = 0) -> FeasibilityReport:
    """assignment.hpp:122-126 / assignment.cpp:264-312, evaluated on the
    device (the first violation and the count; see FeasibilityReport)."""
    return get_solver(device).verify_host(sc, duals, m)


def matching_cost(m: Matching, inst: AssignmentInstance) -> float:
    """core.cpp:95-102: sequential double sum over a ascending."""
    total = 0.0
    for a in range(inst.n_a):
        b = int(m.match_of_a[a])
        if b != K_UNMATCHED:
            total += float(_pair_cost(inst, a, b))
    return total


def _pair_cost(inst: AssignmentInstance, a: int, b: int) -> float:
    if inst.cost is not None:
        return float(inst.cost[a, b])
    if inst.img_a is not None:
        return float(l1_cost(inst.img_a[a:a + 1], inst.img_b[b:b + 1])[0, 0])
    dx = float(inst.pts_a[a, 0]) - float(inst.pts_b[b, 0])
    dy = float(inst.pts_a[a, 1]) - float(inst.pts_b[b, 1])
    return math.sqrt(dx * dx + dy * dy) / math.sqrt(2.0)


def points_threshold_table(eps: float) -> np.ndarray:
    """thr[j] = smallest d2 with scaled_floor(sqrt(d2)/sqrt(2), eps) >= j
    (j = 0..unit_floor+1), so k = searchsorted(thr, d2, 'right') - 1."""
    L = N.lib()
    n = L.otprg_points_threshold_table(float(eps), None, 0)
    if n < 0:
        raise ParameterError("eps must lie in (0, 1)")
    thr = np.empty(n, np.float64)
    L.otprg_points_threshold_table(float(eps), thr.ctypes.data, n)
    return thr


def points_cost(pts_a: np.ndarray, pts_b: np.ndarray) -> np.ndarray:
    """Dense instances.cpp:70-75 cost from point sets (numpy, non-fused)."""
    dx = pts_a[:, None, 0] - pts_b[None, :, 0]
    dy = pts_a[:, None, 1] - pts_b[None, :, 1]
    return np.sqrt(dx * dx + dy * dy) / np.sqrt(2.0)


def gen_uniform_square(n: int, seed: int, dense: bool = False) -> AssignmentInstance:
    """instances.cpp:48-78.  Points come from the reference's mt19937_64
    streams (generated natively by the C ABI); ``dense=True`` also
    materialises the n x n double cost like the reference does."""
    if n < 1:
        raise ParameterError("gen_uniform_square: n must be >= 1")
    pa = np.empty((n, 2), np.float64)
    pb = np.empty((n, 2), np.float64)
    st = N.lib().otprg_uniform_square_points(n, seed, pa.ctypes.data, pb.ctypes.data)
    if st:
        raise ParameterError("gen_uniform_square failed")
    inst = AssignmentInstance(n, n, None, pa, pb, norm_factor=math.sqrt(2.0), seed=seed)
    if dense:
        inst.cost = points_cost(pa, pb)
    return inst


def l1_cost(img_a: np.ndarray, img_b: np.ndarray) -> np.ndarray:
    """Dense load_mnist_pair cost (instances.cpp:114-142): per-image
    normalisation, then sum_p |x_p - y_p| in ascending p, / 2 (host, numpy;
    the sequential sum is kept by accumulating pixel by pixel)."""
    xa = img_a.astype(np.float64) / img_a.astype(np.float64).sum(axis=1, keepdims=True)
    yb = img_b.astype(np.float64) / img_b.astype(np.float64).sum(axis=1, keepdims=True)
    acc = np.zeros((xa.shape[0], yb.shape[0]), np.float64)
    for p in range(xa.shape[1]):
        acc += np.abs(xa[:, p:p + 1] - yb[None, :, p])
    return acc / 2.0


def load_mnist_pair(path: str, n: int, seed: int) -> AssignmentInstance:
    """instances.cpp:80-144: seeded sample of 2n IDX3 images; the first n are A,
    the next n B; cost = L1/2 of the normalised images (computed on the device
    at solve time; norm_factor = 2)."""
    img_a = np.empty((n, 784), np.uint8)
    img_b = np.empty((n, 784), np.uint8)
    err = C.create_string_buffer(256)
    st = N.lib().otprg_load_mnist_pair(path.encode(), n, seed, img_a.ctypes.data,
                                      img_b.ctypes.data, err, 256)
    if st:
        msg = err.value.decode()
        if st == N.PARAMETER:
            raise ParameterError(msg)
        if "magic" in msg or "short" in msg or "truncated" in msg or "dimensions" in msg:
            raise FormatError(msg)
        raise InputError(msg)
    return AssignmentInstance(n, n, None, img_a=img_a, img_b=img_b, norm_factor=2.0, seed=seed)


# ---- optimal transport (include/otpr/ot.hpp) -------------------------------
@dataclass
class OTInstance:
    """ot.hpp:24-37: demand masses mu (A), supply masses nu (B), costs in [0,1]."""
    mu: np.ndarray
    nu: np.ndarray
    cost: np.ndarray
    norm_factor: float = 1.0
    seed: int = 0

    def n_a(self) -> int:
        return len(self.mu)

    def n_b(self) -> int:
        return len(self.nu)

    def renormalize(self) -> None:  # ot.cpp:91-100
        self.mu = self.mu / self.mu.sum()
        self.nu = self.nu / self.nu.sum()


@dataclass
class TransportPlan:
    """core.hpp:150-162 (entries row-major)."""
    a: np.ndarray
    b: np.ndarray
    mass: np.ndarray
    cost: float = 0.0

    def row_sums(self, n_a: int) -> np.ndarray:
        out = np.zeros(n_a)
        for a, m in zip(self.a, self.mass):
            out[a] += m
        return out

    def col_sums(self, n_b: int) -> np.ndarray:
        out = np.zeros(n_b)
        for b, m in zip(self.b, self.mass):
            out[b] += m
        return out

    def total_mass(self) -> float:
        s = 0.0
        for m in self.mass:
            s += float(m)
        return s


@dataclass
class ScaledMasses:
    """ot.hpp:42-49."""
    theta: float
    d: np.ndarray
    s: np.ndarray

    def total_d(self) -> int:
        return int(self.d.sum())

    def total_s(self) -> int:
        return int(self.s.sum())


class _OTProblem(C.Structure):
    _fields_ = [("n_a", C.c_int32), ("n_b", C.c_int32), ("eps", C.c_double),
                ("mu", C.c_void_p), ("nu", C.c_void_p), ("cost", C.c_void_p),
                ("flags", C.c_int32), ("pad", C.c_int32)]


class _OTResult(C.Structure):
    _fields_ = [("ent_a", C.c_void_p), ("ent_b", C.c_void_p), ("ent_mass", C.c_void_p),
                ("entry_cap", C.c_int64), ("free_counts", C.c_void_p), ("free_cap", C.c_int64),
                ("n_entries", C.c_int64), ("cost", C.c_double), ("phases", C.c_int64),
                ("sum_ni", C.c_int64), ("full_match_termination", C.c_int32),
                ("gpu_launches", C.c_int32), ("theta", C.c_double), ("total_d", C.c_int64),
                ("total_s", C.c_int64), ("build_ms", C.c_double), ("loop_ms", C.c_double),
                ("scan_ms", C.c_double), ("solve_ms", C.c_double), ("bytes_touched", C.c_int64)]


def gen_random_ot_rational(n_a: int, n_b: int, seed: int) -> OTInstance:
    """instances.cpp:159-191 (weights 1..50 over their total, u01 costs), renormalised."""
    if n_a < 1 or n_b < 1:
        raise ParameterError("gen_random_ot_rational: sides must be >= 1")
    mu, nu = np.empty(n_a), np.empty(n_b)
    cost = np.empty((n_a, n_b))
    st = N.lib().otprg_random_ot_rational(n_a, n_b, seed, mu.ctypes.data, nu.ctypes.data,
                                          cost.ctypes.data)
    if st:
        raise ParameterError("gen_random_ot_rational failed")
    return OTInstance(mu, nu, cost, seed=seed)


def scale_and_round(inst: OTInstance, eps: float) -> ScaledMasses:
    """ot.cpp:109-128."""
    mu = np.ascontiguousarray(inst.mu, np.float64)
    nu = np.ascontiguousarray(inst.nu, np.float64)
    d, s = np.empty(len(mu), np.int64), np.empty(len(nu), np.int64)
    th = C.c_double()
    st = N.lib().otprg_ot_scale_and_round(len(mu), len(nu), mu.ctypes.data, nu.ctypes.data, eps,
                                          d.ctypes.data, s.ctypes.data, C.byref(th))
    if st:
        raise _STATUS_EXC.get(st, DeviceError)("scale_and_round failed")
    return ScaledMasses(th.value, d, s)


# ---- copy/cluster solver types and hooks (ot.hpp:52-156) --------------------
@dataclass
class CopyInstance:
    """ot.hpp:52-63: rounded costs over the original vertices + copy counts."""
    costs: ScaledCosts
    demand_copies: np.ndarray
    supply_copies: np.ndarray

    def total_demand(self) -> int:
        return int(np.sum(self.demand_copies))

    def total_supply(self) -> int:
        return int(np.sum(self.supply_copies))

    def _c(self):
        k = np.ascontiguousarray(self.costs.k, np.int32)
        d = np.ascontiguousarray(self.demand_copies, np.int64)
        s = np.ascontiguousarray(self.supply_copies, np.int64)
        if k.shape != (len(d), len(s)):
            raise ParameterError("copy counts do not match the cost matrix")
        ci = N.CopyInstance(k.shape[0], k.shape[1], k.ctypes.data, int(self.costs.unit_ceil),
                            d.ctypes.data, s.ctypes.data)
        return ci, (k, d, s)


@dataclass
class DemandCluster:
    """ot.hpp:65-75: copies of a demand vertex at one dual; matched copies as
    flow (b, copies), ascending b."""
    y: int = 0
    free_count: int = 0
    flow: list = field(default_factory=list)

    def matched(self) -> int:
        return sum(c for _, c in self.flow)

    def count(self) -> int:
        return self.free_count + self.matched()


@dataclass
class SupplyCluster:
    """ot.hpp:77-83."""
    y: int = 0
    free_count: int = 0
    matched_count: int = 0

    def count(self) -> int:
        return self.free_count + self.matched_count


@dataclass
class ClusterState:
    """ot.hpp:85-95: per vertex at most two live clusters."""
    demand: list
    supply: list

    def flow_matrix(self, n_a: int, n_b: int) -> np.ndarray:
        f = np.zeros((n_a, n_b), np.int64)
        for a, cs in enumerate(self.demand):
            for c in cs:
                for b, cnt in c.flow:
                    f[a, b] += cnt
        return f

    def free_supply_total(self) -> int:
        return sum(c.free_count for cs in self.supply for c in cs)

    def free_demand_of(self, a: int) -> int:
        return sum(c.free_count for c in self.demand[a])

    def sum_abs_duals(self) -> int:
        return (sum(abs(c.y) * c.count() for cs in self.demand for c in cs)
                + sum(abs(c.y) * c.count() for cs in self.supply for c in cs))

    @staticmethod
    def _from_c(st) -> "ClusterState":
        n_a, n_b = st.n_a, st.n_b

        def arr(ptr, n, ct):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), (n,)).copy() if n else np.zeros(0)

        dem_off = arr(st.dem_off, n_a + 1, C.c_int32)
        nd = int(dem_off[-1])
        dem_y, dem_free = arr(st.dem_y, nd, C.c_int64), arr(st.dem_free, nd, C.c_int64)
        flow_off = arr(st.flow_off, nd + 1, C.c_int64)
        nf = int(flow_off[-1])
        flow_b, flow_cnt = arr(st.flow_b, nf, C.c_int32), arr(st.flow_cnt, nf, C.c_int64)
        sup_off = arr(st.sup_off, n_b + 1, C.c_int32)
        ns = int(sup_off[-1])
        sup_y, sup_free = arr(st.sup_y, ns, C.c_int64), arr(st.sup_free, ns, C.c_int64)
        sup_matched = arr(st.sup_matched, ns, C.c_int64)
        demand = [[DemandCluster(int(dem_y[c]), int(dem_free[c]),
                                 [(int(flow_b[f]), int(flow_cnt[f]))
                                  for f in range(int(flow_off[c]), int(flow_off[c + 1]))])
                   for c in range(int(dem_off[a]), int(dem_off[a + 1]))] for a in range(n_a)]
        supply = [[SupplyCluster(int(sup_y[c]), int(sup_free[c]), int(sup_matched[c]))
                   for c in range(int(sup_off[b]), int(sup_off[b + 1]))] for b in range(n_b)]
        return ClusterState(demand, supply)

    def _c(self):
        dem_off, dem_y, dem_free, flow_off, flow_b, flow_cnt = [0], [], [], [0], [], []
        for cs in self.demand:
            for c in cs:
                dem_y.append(c.y)
                dem_free.append(c.free_count)
                for b, cnt in c.flow:
                    flow_b.append(b)
                    flow_cnt.append(cnt)
                flow_off.append(len(flow_b))
            dem_off.append(len(dem_y))
        sup_off, sup_y, sup_free, sup_matched = [0], [], [], []
        for cs in self.supply:
            for c in cs:
                sup_y.append(c.y)
                sup_free.append(c.free_count)
                sup_matched.append(c.matched_count)
            sup_off.append(len(sup_y))
        keep = [np.asarray(dem_off, np.int32), np.asarray(dem_y, np.int64), np.asarray(dem_free, np.int64),
                np.asarray(flow_off, np.int64), np.asarray(flow_b, np.int32), np.asarray(flow_cnt, np.int64),
                np.asarray(sup_off, np.int32), np.asarray(sup_y, np.int64), np.asarray(sup_free, np.int64),
                np.asarray(sup_matched, np.int64)]
        st = N.ClusterState(len(self.demand), len(self.supply), *[x.ctypes.data for x in keep])
        return st, keep


@dataclass
class ClusterReport:
    """ot.hpp:97-100."""
    violations: list = field(default_factory=list)

    def ok(self) -> bool:
        return not self.violations


def _check_cluster(state: ClusterState, inst: CopyInstance, which: int) -> ClusterReport:
    st, keep = state._c()
    ci, keep2 = inst._c()
    cnt = C.c_int64()
    buf = C.create_string_buffer(1 << 16)
    rc = N.lib().otprg_check_cluster_state(C.byref(st), C.byref(ci), which, C.byref(cnt), buf, len(buf))
    if rc:
        raise ParameterError("cluster state does not match the copy instance")
    msgs = buf.value.decode().split("\n") if cnt.value else []
    return ClusterReport(msgs[: cnt.value])


def check_cluster_invariant(state: ClusterState, inst: CopyInstance) -> ClusterReport:
    """ot.hpp:102-107 / ot.cpp:190-265."""
    return _check_cluster(state, inst, 0)


def check_cluster_feasibility(state: ClusterState, inst: CopyInstance) -> ClusterReport:
    """ot.hpp:109-113 / ot.cpp:267-315."""
    return _check_cluster(state, inst, 1)


@dataclass
class ClusterPhaseSnapshot:
    """ot.hpp:115-122 (a copy: valid after the callback too)."""
    phase: int
    inst: CopyInstance
    state: ClusterState
    n_i: int
    sum_abs_before: int
    sum_abs_after: int


@dataclass
class ClusterOptions:
    """ot.hpp:124-129 (and OTOptions, ot.hpp:153-156): after every phase the
    greedy-maximality / cluster-invariant / feasibility checks (host), and an
    observer called with a ClusterPhaseSnapshot."""
    check_invariants: bool = False
    observer: Optional[Callable] = None


OTOptions = ClusterOptions


@dataclass
class ClusterSolveResult:
    """ot.hpp:131-135: final state before completion, flow with completion."""
    state: ClusterState
    flow: np.ndarray
    stats: SolveStats


def _c_options(opt: Optional[ClusterOptions]):
    """(N.OTOptions or None, the callback keep-alive, the error box)."""
    if opt is None or (not opt.check_invariants and opt.observer is None):
        return None, None, None
    err = []
    cb = N.CLUSTER_OBSERVER()  # NULL
    if opt.observer is not None:
        cache = {}

        def _obs(snap_p, _user):
            try:
                sn = snap_p.contents
                if "inst" not in cache:  # the copy instance does not change between phases
                    ci = sn.inst
                    k = np.ctypeslib.as_array(C.cast(ci.k, C.POINTER(C.c_int32)), (ci.n_a, ci.n_b)).copy()
                    d = np.ctypeslib.as_array(C.cast(ci.demand_copies, C.POINTER(C.c_int64)), (ci.n_a,)).copy()
                    s = np.ctypeslib.as_array(C.cast(ci.supply_copies, C.POINTER(C.c_int64)), (ci.n_b,)).copy()
                    cache["inst"] = CopyInstance(ScaledCosts(0.0, k, int(ci.unit_ceil), int(ci.unit_ceil)), d, s)
                opt.observer(ClusterPhaseSnapshot(int(sn.phase), cache["inst"], ClusterState._from_c(sn.state),
                                                  int(sn.n_i), int(sn.sum_abs_before), int(sn.sum_abs_after)))
                return 0
            except BaseException as e:  # re-raised by the caller after the C call returns
                err.append(e)
                return 1

        cb = N.CLUSTER_OBSERVER(_obs)
    o = N.OTOptions(int(bool(opt.check_invariants)), 0, cb, None)
    return o, cb, err


def _raise_opts(solver, st: int, err):
    if st == N.ABORTED and err:
        raise err[0]
    solver._raise(st)


def solve_copy_matching(inst: CopyInstance, eps: float, opt: Optional[ClusterOptions] = None,
                        device: int = 0) -> ClusterSolveResult:
    """ot.hpp:135-141 / ot.cpp:418-637 on the device (admissible-cluster
    scans) with the claim step and cluster bookkeeping on the host."""
    ci, keep = inst._c()
    n_a, n_b = ci.n_a, ci.n_b
    solver = get_solver(device)
    o, cb, err = _c_options(opt)
    fcap = min(SolveStats.phase_bound(eps) + 16, N.MAX_PHASES + 2) if 0.0 < eps < 1.0 else 16
    fc = np.zeros(fcap, np.int64)
    flow = np.zeros((n_a, n_b), np.int64)
    r = N.CopyResult(flow.ctypes.data, fc.ctypes.data, fcap, 0, 0, 0, 0)
    st = solver._L.otprg_solve_copy_matching(solver._ctx, C.byref(ci), float(eps),
                                             C.byref(o) if o is not None else None, C.byref(r))
    if st:
        _raise_opts(solver, st, err)
    cs = N.ClusterState()
    st = solver._L.otprg_copy_state(solver._ctx, C.byref(cs))
    if st:
        solver._raise(st)
    stats = SolveStats(phases=int(r.phases), free_counts=fc[: r.phases].copy(), sum_ni=int(r.sum_ni),
                       full_match_termination=bool(r.full_match_termination),
                       device=dict(gpu_launches=int(r.gpu_launches)))
    return ClusterSolveResult(ClusterState._from_c(cs), flow, stats)


def plan_from_flow(flow: np.ndarray, sm: ScaledMasses, inst: OTInstance) -> TransportPlan:
    """ot.hpp:143-151 / ot.cpp:639-703 (host, the reference's FP64 order)."""
    mu = np.ascontiguousarray(inst.mu, np.float64)
    nu = np.ascontiguousarray(inst.nu, np.float64)
    cost = np.ascontiguousarray(inst.cost, np.float64)
    f = np.ascontiguousarray(flow, np.int64)
    if f.shape != (len(mu), len(nu)) or cost.shape != f.shape:
        raise ParameterError("flow matrix dimensions do not match the instance")
    p = _OTProblem(len(mu), len(nu), 0.5, mu.ctypes.data, nu.ctypes.data, cost.ctypes.data, 0, 0)
    cap = int(np.count_nonzero(f)) + len(mu) + len(nu) + 16
    while True:
        ea, eb, em = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap)
        r = _OTResult()
        r.ent_a, r.ent_b, r.ent_mass, r.entry_cap = ea.ctypes.data, eb.ctypes.data, em.ctypes.data, cap
        d = np.ascontiguousarray(sm.d, np.int64)
        s = np.ascontiguousarray(sm.s, np.int64)
        st = N.lib().otprg_plan_from_flow(C.byref(p), f.ctypes.data, float(sm.theta), d.ctypes.data,
                                          s.ctypes.data, C.byref(r))
        if st:
            raise _STATUS_EXC.get(st, DeviceError)("plan_from_flow failed")
        if r.n_entries <= cap:
            break
        cap = int(r.n_entries)
    ne = int(r.n_entries)
    return TransportPlan(ea[:ne].copy(), eb[:ne].copy(), em[:ne].copy(), float(r.cost))


def last_cluster_state(device: int = 0) -> ClusterState:
    """ClusterSolveResult::state of the last solve_ot / solve_copy_matching on
    this device's shared solver (the state before completion)."""
    solver = get_solver(device)
    cs = N.ClusterState()
    st = solver._L.otprg_copy_state(solver._ctx, C.byref(cs))
    if st:
        solver._raise(st)
    return ClusterState._from_c(cs)


def solve_ot(inst: OTInstance, eps: float, opt: Optional[OTOptions] = None, device: int = 0):
    """ot.hpp:161-163 / ot.cpp:705-732 -> (TransportPlan, SolveStats)."""
    mu = np.ascontiguousarray(inst.mu, np.float64)
    nu = np.ascontiguousarray(inst.nu, np.float64)
    cost = np.ascontiguousarray(inst.cost, np.float64)
    if cost.shape != (len(mu), len(nu)):
        raise ParameterError("OT cost matrix dimensions do not match mass vectors")
    solver = get_solver(device)
    p = _OTProblem(len(mu), len(nu), float(eps), mu.ctypes.data, nu.ctypes.data, cost.ctypes.data,
                   0, 0)
    o, cb, err = _c_options(opt)
    cap = 4 * (len(mu) + len(nu)) + 64
    if o is not None:  # hooks run once: room for any plan (debug sizes)
        cap = max(cap, len(mu) * len(nu))
    fcap = (min(SolveStats.phase_bound(eps / 3.0) + 16, N.MAX_PHASES + 2)
            if 0.0 < eps < 1.0 else 16)  # C ABI validates eps
    ea, eb, em = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap)
    fc = np.zeros(fcap, np.int64)
    r = _OTResult()
    r.ent_a, r.ent_b, r.ent_mass, r.entry_cap = ea.ctypes.data, eb.ctypes.data, em.ctypes.data, cap
    r.free_counts, r.free_cap = fc.ctypes.data, fcap
    st = solver._L.otprg_solve_ot_opts(solver._ctx, C.byref(p), C.byref(o) if o is not None else None,
                                       C.byref(r))
    if st:
        _raise_opts(solver, st, err)
    if r.n_entries > cap:  # rerun with room for every entry
        cap = int(r.n_entries)
        ea, eb, em = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap)
        r.ent_a, r.ent_b, r.ent_mass, r.entry_cap = ea.ctypes.data, eb.ctypes.data, em.ctypes.data, cap
        st = solver._L.otprg_solve_ot(solver._ctx, C.byref(p), C.byref(r))
        if st:
            solver._raise(st)
    ne = int(r.n_entries)
    plan = TransportPlan(ea[:ne].copy(), eb[:ne].copy(), em[:ne].copy(), float(r.cost))
    stats = SolveStats(phases=int(r.phases), free_counts=fc[: r.phases].copy(), sum_ni=int(r.sum_ni),
                       full_match_termination=bool(r.full_match_termination),
                       device=dict(theta=r.theta, total_d=int(r.total_d), total_s=int(r.total_s),
                                   build_ms=r.build_ms, loop_ms=r.loop_ms, scan_ms=r.scan_ms,
                                   solve_ms=r.solve_ms, bytes_touched=int(r.bytes_touched),
                                   gpu_launches=int(r.gpu_launches)))
    return plan, stats


# ---- Sinkhorn baseline (sinkhorn.hpp:13-31) ------------
@dataclass
class SinkhornConfig:
    """sinkhorn.hpp:13-18."""
    reg: float = 0.01
    max_iters: int = 10000
    tol: float = 1e-9
    time_budget_ms: float = 0.0


@dataclass
class SinkhornResult:
    """sinkhorn.hpp:20-26 (plan rounded to exact marginals), plus device timings."""
    plan: Optional[TransportPlan]
    iters: int
    cost: float
    converged: bool
    marginal_violation: float
    device: dict = field(default_factory=dict)


class _SkConfig(C.Structure):
    _fields_ = [("reg", C.c_double), ("max_iters", C.c_int32), ("pad", C.c_int32),
                ("tol", C.c_double), ("time_budget_ms", C.c_double)]


class _SkResult(C.Structure):
    _fields_ = [("ent_a", C.c_void_p), ("ent_b", C.c_void_p), ("ent_mass", C.c_void_p),
                ("entry_cap", C.c_int64), ("n_entries", C.c_int64), ("cost", C.c_double),
                ("iters", C.c_int32), ("converged", C.c_int32), ("marginal_violation", C.c_double),
                ("build_ms", C.c_double), ("loop_ms", C.c_double), ("round_ms", C.c_double)]


def reg_for_eps(eps: float, n: int) -> float:
    """bench.cpp:38-41: reg = eps / (4 ln n), n clamped to >= 2."""
    return eps / (4.0 * math.log(max(float(n), 2.0)))


def sinkhorn(inst: OTInstance, cfg: SinkhornConfig, device: int = 0,
             entries: bool = True) -> SinkhornResult:
    """sinkhorn.hpp:28-31 / sinkhorn.cpp:69-151 on the device (FP64).
    ``entries=False`` skips the D2H of the dense plan (cost and counts only)."""
    mu = np.ascontiguousarray(inst.mu, np.float64)
    nu = np.ascontiguousarray(inst.nu, np.float64)
    cost = np.ascontiguousarray(inst.cost, np.float64)
    if cost.shape != (len(mu), len(nu)):
        raise ParameterError("OT cost matrix dimensions do not match mass vectors")
    solver = get_solver(device)
    p = _OTProblem(len(mu), len(nu), 0.5, mu.ctypes.data, nu.ctypes.data, cost.ctypes.data, 0, 0)
    c = _SkConfig(float(cfg.reg), int(cfg.max_iters), 0, float(cfg.tol), float(cfg.time_budget_ms))
    r = _SkResult()
    st = solver._L.otprg_sinkhorn(solver._ctx, C.byref(p), C.byref(c), C.byref(r))
    if st:
        solver._raise(st)
    plan = None
    if entries:
        ne = int(r.n_entries)
        ea, eb, em = np.empty(max(ne, 1), np.int32), np.empty(max(ne, 1), np.int32), np.empty(max(ne, 1))
        r2 = _SkResult()
        r2.ent_a, r2.ent_b, r2.ent_mass, r2.entry_cap = ea.ctypes.data, eb.ctypes.data, em.ctypes.data, ne
        st = solver._L.otprg_sinkhorn(solver._ctx, C.byref(p), C.byref(c), C.byref(r2))
        if st:
            solver._raise(st)
        plan = TransportPlan(ea[:ne].copy(), eb[:ne].copy(), em[:ne].copy(), float(r2.cost))
        r = r2
    return SinkhornResult(plan, int(r.iters), float(r.cost), bool(r.converged),
                          float(r.marginal_violation),
                          device=dict(build_ms=r.build_ms, loop_ms=r.loop_ms, round_ms=r.round_ms,
                                      n_entries=int(r.n_entries)))
