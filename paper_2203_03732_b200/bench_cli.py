"""GPU benchmark CLI with the reference's CSV schema and exit codes (SURVEY
§8(f) rank 2): a drop-in for ``otbench`` (tools/otbench.cpp) on the solvers
this library provides.

    python -m paper_2203_03732_b200.bench_cli gen   --n 1000 --seed 1 --out inst.bin
    python -m paper_2203_03732_b200.bench_cli solve --solver pushrelabel --n 1000 --eps 0.1 [--verify]
    python -m paper_2203_03732_b200.bench_cli bench --solvers pushrelabel --n 500 1000 --eps 0.1 0.01

* ``run_solver`` mirrors bench.cpp:44-199: same RunRecord fields, the same
  timing boundary (the whole solve incl. cost rounding; instance generation
  and verification outside the timer), the same ``--verify`` checks (per phase:
  verify_feasibility, matched-set monotonicity, dual progress, greedy
  maximality; phase / Σn_i bounds; ``pushrelabel-ot``: a rerun with
  OTOptions::check_invariants), ``--no-normalize`` semantics.  The
  solvers ``pushrelabel``, ``pushrelabel-ot`` and ``sinkhorn`` run on the GPU
  through this package; the exact oracles ``hungarian`` and ``exact-ot`` are
  not on the device path (ParameterError, exit 2), so the oracle-gap check of
  ``--verify`` is reported as a note.
* CSV: ``csv_header`` / ``csv_row`` / ``write_csv`` / ``aggregate`` /
  ``write_aggregate_csv`` (bench.cpp:210-266) with ``format_double`` = C++
  ``std::to_chars`` shortest form (bench.cpp:203-208).
* Instance cache: ``save_instance`` / ``load_instance`` in the reference's
  binary format (instances.cpp:195-246, magic ``OTPRINS1``).
* Exit codes (otbench.cpp:187-209): 0 ok, 2 parameter, 3 input/format,
  4 numerical, 5 invariant violation (``--verify``), 1 other.
"""
from __future__ import annotations

import argparse
import decimal
import math
import os
import struct
import sys
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import api as A

_MAGIC = b"OTPRINS1"


# ---- number formatting (bench.cpp:203-208) ----------------------------------
def format_double(v: float) -> str:
    """std::to_chars(double) shortest form: the shortest round-trip digits,
    printed fixed or scientific, whichever is shorter (fixed on a tie)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    t = decimal.Decimal(repr(abs(v))).normalize().as_tuple() if v != 0 else None
    if t is None:
        return sign + "0"
    digits = "".join(map(str, t.digits))
    exp = t.exponent  # value = digits * 10**exp
    # fixed
    if exp >= 0:
        fixed = digits + "0" * exp
    else:
        point = len(digits) + exp
        fixed = (digits[:point] + "." + digits[point:]) if point > 0 else \
            "0." + "0" * (-point) + digits
    # scientific d.ddde±XX
    e10 = len(digits) - 1 + exp
    mant = digits[0] + ("." + digits[1:] if len(digits) > 1 else "")
    sci = f"{mant}e{'-' if e10 < 0 else '+'}{abs(e10):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


# ---- records and CSV (bench.hpp:18-82, bench.cpp:210-266) -------------------
@dataclass
class RunRecord:
    solver: str
    n: int = 0
    eps: Optional[float] = None
    reg: Optional[float] = None
    seed: int = 0
    cost: float = 0.0
    oracle_cost: Optional[float] = None
    time_ms: float = 0.0
    phases: int = 0


@dataclass
class SolveRequest:
    solver: str
    eps: float = 0.1
    reg: Optional[float] = None
    threads: int = 1
    verify: bool = False
    no_normalize: bool = False
    sinkhorn_max_iters: int = 10000
    device: int = 0


@dataclass
class SolveOutcome:
    record: RunRecord
    verify_violations: list = field(default_factory=list)
    notes: list = field(default_factory=list)


def csv_header() -> str:
    return "solver,n,eps,reg,seed,cost,oracle_cost,time_ms,phases"


def csv_row(r: RunRecord) -> str:
    f = format_double
    return ",".join([r.solver, str(r.n), f(r.eps) if r.eps is not None else "",
                     f(r.reg) if r.reg is not None else "", str(r.seed), f(r.cost),
                     f(r.oracle_cost) if r.oracle_cost is not None else "", f(r.time_ms),
                     str(r.phases)])


def write_csv(path: str, rows: list) -> None:
    try:
        with open(path, "w") as out:
            out.write(csv_header() + "\n")
            for r in rows:
                out.write(csv_row(r) + "\n")
    except OSError as e:
        raise A.InputError(f"cannot open for writing: {path}") from e


def aggregate(rows: list) -> list:
    cells = {}
    for r in rows:
        key = (r.solver, r.n, r.eps if r.eps is not None else -1.0)
        c = cells.setdefault(key, {"solver": r.solver, "n": r.n, "eps": r.eps, "runs": 0,
                                   "mean_cost": 0.0, "mean_time_ms": 0.0})
        c["runs"] += 1
        c["mean_cost"] += r.cost
        c["mean_time_ms"] += r.time_ms
    out = []
    for key in sorted(cells):  # std::map order over (solver, n, eps)
        c = cells[key]
        c["mean_cost"] /= c["runs"]
        c["mean_time_ms"] /= c["runs"]
        out.append(c)
    return out


def write_aggregate_csv(path: str, rows: list) -> None:
    try:
        with open(path, "w") as out:
            out.write("solver,n,eps,runs,mean_cost,mean_time_ms\n")
            for r in rows:
                eps = format_double(r["eps"]) if r["eps"] is not None else ""
                out.write(f"{r['solver']},{r['n']},{eps},{r['runs']},"
                          f"{format_double(r['mean_cost'])},{format_double(r['mean_time_ms'])}\n")
    except OSError as e:
        raise A.InputError(f"cannot open for writing: {path}") from e


# ---- instance cache (instances.cpp:195-246) --------------------------------
def save_instance(inst: A.AssignmentInstance, path: str) -> None:
    inst.validate()
    cost = np.ascontiguousarray(inst.dense_cost(), np.float64)
    try:
        with open(path, "wb") as out:
            out.write(_MAGIC)
            out.write(struct.pack("<IIdQ", inst.n_a, inst.n_b, inst.norm_factor, inst.seed))
            out.write(cost.tobytes())
    except OSError as e:
        raise A.InputError(f"cannot open for writing: {path}") from e


def load_instance(path: str) -> A.AssignmentInstance:
    try:
        f = open(path, "rb")
    except OSError as e:
        raise A.InputError(f"cannot open instance file: {path}") from e
    with f:
        if f.read(8) != _MAGIC:
            raise A.FormatError(f"not an instance cache file: {path}")
        hdr = f.read(24)
        if len(hdr) != 24:
            raise A.FormatError(f"corrupt instance header: {path}")
        n_a, n_b, norm, seed = struct.unpack("<IIdQ", hdr)
        if n_a == 0 or n_b == 0:
            raise A.FormatError(f"corrupt instance header: {path}")
        raw = f.read(8 * n_a * n_b)
        if len(raw) != 8 * n_a * n_b:
            raise A.FormatError(f"instance payload truncated: {path}")
    cost = np.frombuffer(raw, np.float64).reshape(n_a, n_b).copy()
    return A.AssignmentInstance(n_a, n_b, cost, norm_factor=norm, seed=seed)


# ---- run_solver (bench.cpp:44-199) ------------------------------------------
def _verify_observer(out: SolveOutcome, device: int):
    prev = {"matched": 0}

    def obs(snap: A.PhaseSnapshot):
        rep = A.get_solver(device).verify_feasibility()  # the snapshot's (live) device state
        for v in rep.violations:
            out.verify_violations.append(f"phase {snap.phase}: {v}")
        matched = snap.matching.size()
        if matched < prev["matched"]:
            out.verify_violations.append(f"phase {snap.phase}: matched demand count decreased")
        prev["matched"] = matched
        if snap.sum_abs_after - snap.sum_abs_before < len(snap.workset.b_free):
            out.verify_violations.append(
                f"phase {snap.phase}: dual magnitude progress below the free count")
        prime_a = {a for a, _ in snap.workset.m_prime}
        prime_b = {b for _, b in snap.workset.m_prime}
        for i, b in enumerate(snap.workset.b_free):
            if int(b) in prime_b:
                continue
            for a in snap.workset.e_admissible[i]:
                if int(a) not in prime_a:
                    out.verify_violations.append(
                        f"phase {snap.phase}: greedy matching left an admissible pair unmatched")

    return obs


_warmed: set = set()


def _warm_up(device: int) -> None:
    """Context creation, module loading and first-touch allocations happen
    once per process, outside the timer (the reference, a CPU library, has
    nothing to initialise; a long-lived GPU library amortises this)."""
    if device in _warmed:
        return
    rng = np.random.default_rng(0)
    cost = rng.random((8, 8))
    A.solve_assignment(A.AssignmentInstance(8, 8, cost), A.AssignmentOptions(eps=0.1, device=device))
    A.solve_ot(A.OTInstance(np.full(8, 0.125), np.full(8, 0.125), cost), 0.1, device=device)
    _warmed.add(device)


# The GPU solver names SURVEY §8(b) proposes for a GPU-aware run_solver; they
# run the same device paths as the reference's own names (and keep their own
# name in the CSV).
ALIASES = {"pushrelabel-gpu": "pushrelabel", "pushrelabel-ot-gpu": "pushrelabel-ot",
           "sinkhorn-gpu": "sinkhorn"}


def run_solver(inst: A.AssignmentInstance, req: SolveRequest) -> SolveOutcome:
    inst.validate()
    rec = RunRecord(req.solver, n=min(inst.n_a, inst.n_b), seed=inst.seed)
    out = SolveOutcome(rec)
    scale = inst.norm_factor if req.no_normalize else 1.0
    eps = req.eps / inst.norm_factor if req.no_normalize else req.eps
    m_side = min(inst.n_a, inst.n_b)
    solver = ALIASES.get(req.solver, req.solver)

    if solver == "pushrelabel":
        rec.eps = req.eps
        opt = A.AssignmentOptions(eps=eps, threads=req.threads, device=req.device)
        _warm_up(req.device)
        t0 = time.perf_counter()
        m, st = A.solve_assignment(inst, opt)
        rec.time_ms = (time.perf_counter() - t0) * 1e3
        rec.cost = A.matching_cost(m, inst) * scale
        rec.phases = st.phases
        if req.verify:  # untimed checked rerun (deterministic)
            vopt = A.AssignmentOptions(eps=eps, device=req.device, observer=_verify_observer(out, req.device))
            vm, vs = A.solve_assignment(inst, vopt)
            if vs.phases > A.SolveStats.phase_bound(eps):
                out.verify_violations.append("phase count exceeds bound")
            if vs.sum_ni > A.SolveStats.sum_ni_bound(eps, m_side):
                out.verify_violations.append("total free count exceeds bound")
            if vs.full_match_termination:
                out.notes.append("terminated by full matching")
            out.notes.append("oracle gap not checked: hungarian is not on the device path")
        return out

    if solver == "pushrelabel-ot":
        if inst.n_a != inst.n_b:
            raise A.InputError("assignment_to_ot needs a balanced instance")
        rec.eps = req.eps
        _warm_up(req.device)
        cost = np.ascontiguousarray(inst.dense_cost(), np.float64)
        ot = A.OTInstance(np.full(inst.n_a, 1.0 / inst.n_a), np.full(inst.n_b, 1.0 / inst.n_b),
                          cost, norm_factor=inst.norm_factor, seed=inst.seed)  # assignment_to_ot
        t0 = time.perf_counter()
        plan, st = A.solve_ot(ot, eps, device=req.device)
        rec.time_ms = (time.perf_counter() - t0) * 1e3
        rec.cost = plan.cost * scale
        rec.phases = st.phases
        if req.verify:  # bench.cpp:141-156: an untimed rerun with OTOptions::check_invariants
            try:
                A.solve_ot(ot, eps, A.OTOptions(check_invariants=True), device=req.device)
            except A.InvariantViolation as err:
                out.verify_violations.append(str(err))
            out.notes.append("oracle gap not checked: exact-ot is not on the device path")
        return out

    if solver == "sinkhorn":
        if inst.n_a != inst.n_b:
            raise A.InputError("assignment_to_ot needs a balanced instance")
        rec.eps = req.eps
        _warm_up(req.device)
        cost = np.ascontiguousarray(inst.dense_cost(), np.float64)
        ot = A.OTInstance(np.full(inst.n_a, 1.0 / inst.n_a), np.full(inst.n_b, 1.0 / inst.n_b),
                          cost, norm_factor=inst.norm_factor, seed=inst.seed)
        cfg = A.SinkhornConfig(reg=req.reg if req.reg is not None else
                               A.reg_for_eps(eps, max(inst.n_a, inst.n_b)),
                               max_iters=req.sinkhorn_max_iters)
        rec.reg = cfg.reg
        t0 = time.perf_counter()
        res = A.sinkhorn(ot, cfg, device=req.device, entries=False)  # the cost is computed on the device
        rec.time_ms = (time.perf_counter() - t0) * 1e3
        rec.cost = res.cost * scale
        rec.phases = res.iters
        if not res.converged:
            out.notes.append("sinkhorn stopped before tolerance (violation "
                             f"{format_double(res.marginal_violation)})")
        if req.verify:
            out.notes.append("exact-ot gap not checked: exact-ot is not on the device path")
        return out

    if req.solver in ("hungarian", "exact-ot"):
        raise A.ParameterError(f"solver not provided by the device library: {req.solver}")
    raise A.ParameterError(f"unknown solver: {req.solver}")


# ---- CLI (otbench.cpp) -------------------------------------------------------
def _make_instance(args) -> A.AssignmentInstance:
    if getattr(args, "input", None):
        return load_instance(args.input)
    if args.kind == "square":
        return A.gen_uniform_square(args.n, args.seed)
    images = args.images or os.environ.get("OTPR_DATA")
    if not images:
        raise A.ParameterError("--kind mnist needs --images (or $OTPR_DATA)")
    return A.load_mnist_pair(images, args.n, args.seed)


def _print_outcome(o: SolveOutcome) -> None:
    r = o.record
    s = f"solver={r.solver} n={r.n}"
    if r.eps is not None:
        s += f" eps={format_double(r.eps)}"
    if r.reg is not None:
        s += f" reg={format_double(r.reg)}"
    s += f" seed={r.seed} cost={format_double(r.cost)}"
    if r.oracle_cost is not None:
        s += f" oracle_cost={format_double(r.oracle_cost)}"
    s += f" time_ms={format_double(r.time_ms)} phases={r.phases}"
    print(s)
    for n in o.notes:
        print(f"note: {n}")
    for v in o.verify_violations:
        print(f"violation: {v}")


def _instance_flags(p):
    p.add_argument("--in", dest="input", default="")
    p.add_argument("--kind", default="square", choices=["square", "mnist"])
    p.add_argument("--images", default="")
    p.add_argument("--n", type=int, default=100)
    p.add_argument("--seed", type=int, default=1)


def _run(argv) -> int:
    ap = argparse.ArgumentParser(prog="otbench-gpu",
                                 description="approximate optimal transport / assignment benchmark")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="generate and cache an instance")
    _instance_flags(g)
    g.add_argument("--out", required=True)
    s = sub.add_parser("solve", help="run one solver on one instance")
    _instance_flags(s)
    s.add_argument("--solver", required=True,
                   choices=["pushrelabel", "pushrelabel-ot", "sinkhorn", "hungarian", "exact-ot"] + list(ALIASES))
    s.add_argument("--eps", type=float, default=0.1)
    s.add_argument("--reg", type=float, default=None)
    s.add_argument("--threads", type=int, default=1)
    s.add_argument("--sinkhorn-max-iters", type=int, default=10000)
    s.add_argument("--verify", action="store_true")
    s.add_argument("--no-normalize", action="store_true")
    s.add_argument("--csv", default="")
    b = sub.add_parser("bench", help="sweep a (solver, n, eps) grid")
    b.add_argument("--solvers", nargs="+", default=["pushrelabel", "sinkhorn"])
    b.add_argument("--n", nargs="+", type=int, default=[500, 1000, 2000])
    b.add_argument("--eps", nargs="+", type=float, default=[0.1, 0.01])
    b.add_argument("--runs", type=int, default=30)
    b.add_argument("--seed0", type=int, default=1)
    b.add_argument("--kind", default="square", choices=["square", "mnist"])
    b.add_argument("--images", default="")
    b.add_argument("--out", default="bench.csv")
    b.add_argument("--aggregate", default="")
    b.add_argument("--threads", type=int, default=1)
    b.add_argument("--no-normalize", action="store_true")
    b.add_argument("--sinkhorn-max-iters", type=int, default=10000)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # CLI11 parse errors exit with 105; argparse uses 2
        return int(e.code or 0)

    if args.cmd == "gen":
        inst = _make_instance(args)
        save_instance(inst, args.out)
        print(f"wrote {args.out}: n_a={inst.n_a} n_b={inst.n_b} seed={inst.seed} "
              f"norm_factor={format_double(inst.norm_factor)}")
        return 0
    if args.cmd == "solve":
        req = SolveRequest(args.solver, args.eps, args.reg, args.threads, args.verify,
                           args.no_normalize, args.sinkhorn_max_iters)
        o = run_solver(_make_instance(args), req)
        _print_outcome(o)
        if args.csv:
            write_csv(args.csv, [o.record])
        return 5 if o.verify_violations else 0
    rows = []
    for solver in args.solvers:
        for n in args.n:
            for eps in args.eps:
                for run_id in range(args.runs):
                    ns = argparse.Namespace(input="", kind=args.kind, images=args.images, n=n,
                                            seed=args.seed0 + run_id)
                    req = SolveRequest(solver, eps, None, args.threads, False, args.no_normalize,
                                       args.sinkhorn_max_iters)
                    rows.append(run_solver(_make_instance(ns), req).record)
    write_csv(args.out, rows)
    print(f"wrote {len(rows)} rows to {args.out}")
    if args.aggregate:
        write_aggregate_csv(args.aggregate, aggregate(rows))
        print(f"wrote aggregates to {args.aggregate}")
    return 0


def main(argv=None) -> int:
    try:
        return _run(sys.argv[1:] if argv is None else argv)
    except A.ParameterError as e:
        print(f"parameter error: {e}", file=sys.stderr)
        return 2
    except A.FormatError as e:
        print(f"format error: {e}", file=sys.stderr)
        return 3
    except A.InputError as e:
        print(f"input error: {e}", file=sys.stderr)
        return 3
    except A.NumericalError as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return 4
    except A.InvariantViolation as e:
        print(f"invariant violation: {e}", file=sys.stderr)
        return 5
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
