"""A-row-sharded assignment solve over several GPUs.

Rank g owns the demand range [bounds[g], bounds[g+1]) of every rounded-cost
row (its slab of kT, built on its GPU from the point sets); the matching,
the integer duals and the deferred-acceptance holders are replicated, and
every rank runs the same deterministic phase, so only candidate lists cross
NVLink.  Per phase (reference: solve_oriented, assignment.cpp:316-364):

    top      apply the previous M', termination test      (every rank)
    scan     first K admissible a >= start of every free b in the slab
    gather   all-gather of the per-rank candidate slots   (NCCL / NVLink)
    DA       deferred acceptance over the merged lists; chains that reach
             a truncated slab park -> rescan -> gather -> resume

Results are bit-identical for every shard count (and to the single-GPU
solver / the reference): the merged candidate order is the row order and
deferred acceptance with a common priority has one outcome.

Backends (same driver): ``DeviceRank`` drives one otprg_ctx through the C
ABI; the exchange is ``LocalExchange`` (all ranks in one process share one
buffer: several logical shards on one GPU) or ``TorchDistExchange`` (one
process per GPU, torch.distributed all_gather over NCCL).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .api import AssignmentInstance, AssignmentOptions, ParameterError, Solver, _check_options

K_DEFAULT = 16


class DeviceRank:
    """One shard: an otprg_ctx prepared with the slab [lo, hi)."""

    def __init__(self, device: int = 0):
        self.solver = Solver(device)
        self._L, self._ctx = self.solver._L, self.solver._ctx

    def _ok(self, st):
        if st:
            self.solver._raise(st)

    def prepare(self, inst: AssignmentInstance, eps: float, n_shards: int, shard: int,
                K: int = K_DEFAULT, storage: str = "auto", on_the_fly: bool = False) -> np.ndarray:
        p = self.solver._problem(inst, eps, storage)
        if on_the_fly:  # no kT slab: scans compute k from the points (threshold table)
            from . import _native as N
            p.flags |= N.FLAG_ON_THE_FLY
        bounds = np.zeros(n_shards + 1, np.int32)
        self._ok(self._L.otprg_shard_prepare(self._ctx, C.byref(p), n_shards, shard, K,
                                             bounds.ctypes.data))
        self.n_shards, self.shard, self.K = n_shards, shard, K
        self.cap = min(inst.n_a, inst.n_b)
        self.shape = (inst.n_a, inst.n_b, eps)
        self.bounds = bounds
        return bounds

    def begin(self):
        self._ok(self._L.otprg_shard_begin(self._ctx))

    def top(self) -> tuple[int, bool]:
        n, fin = C.c_int32(), C.c_int32()
        self._ok(self._L.otprg_shard_top(self._ctx, C.byref(n), C.byref(fin)))
        return int(n.value), bool(fin.value)

    def scan(self, cand_ptr: int, meta_ptr: int, cap: int, refill: bool):
        self._ok(self._L.otprg_shard_scan(self._ctx, cand_ptr, meta_ptr, cap, int(refill)))

    def da(self, cand_ptr: int, meta_ptr: int, cap: int, resume: bool) -> int:
        parked = C.c_int32()
        self._ok(self._L.otprg_shard_da(self._ctx, cand_ptr, meta_ptr, cap, int(resume),
                                        C.byref(parked)))
        return int(parked.value)

    def snapshot(self):
        """The replicated state before completion (otprg_snapshot): matching
        (caller orientation), duals (internal), phases, free_counts."""
        n_a, n_b, eps = self.shape
        r, bufs = self.solver._result(n_a, n_b, eps)
        self._ok(self._L.otprg_snapshot(self._ctx, C.byref(r)))
        return Solver._pack(r, bufs)

    def finish(self):
        n_a, n_b, eps = self.shape
        r, bufs = self.solver._result(n_a, n_b, eps)
        self._ok(self._L.otprg_shard_finish(self._ctx, C.byref(r)))
        return Solver._pack(r, bufs)

    def set_stream(self, stream_handle: int):
        self._ok(self._L.otprg_set_stream(self._ctx, stream_handle))

    def close(self):
        self._L.otprg_set_stream(self._ctx, None)
        self.solver.close()


def _buffers(n_shards: int, cap: int, K: int, device: int):
    import torch
    cand = torch.full((n_shards * cap * K,), -1, dtype=torch.int32, device=f"cuda:{device}")
    meta = torch.zeros((n_shards * cap * 2,), dtype=torch.int32, device=f"cuda:{device}")
    return cand, meta


class LocalExchange:
    """All ranks in this process write their slots into one shared buffer."""

    def gather(self, n, *args):
        return None


class TorchDistExchange:
    """One process per GPU: all_gather of the rank slots (NCCL over NVLink).
    Only the used prefix moves: with n proposers in the phase the kernels
    index the buffers as [world][n][K] / [world][n][2]."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def gather(self, n, cand=None, meta=None, K=0):
        import torch.distributed as dist
        for t, per in ((cand, n * K), (meta, n * 2)):
            if t is None:
                continue
            view = t.narrow(0, 0, self.world * per)
            mine = view.narrow(0, self.rank * per, per).clone()
            if t.is_cuda and dist.get_backend() == "nccl":
                dist.all_gather_into_tensor(view, mine)
            else:  # gloo (CPU tests of the protocol; one-GPU multi-process checks)
                dist.all_gather(list(view.split(per)), mine)
        # (CUDA: the collective is ordered on the current stream, which the
        # contexts share — otprg_set_stream — so the DA launch follows it
        # without a host sync)


def run_phases(ranks, exchange, cand_ptr, meta_ptr, cap: int, gather_args=()):
    """The per-phase protocol over the ranks this process drives (one rank per
    process with TorchDistExchange; every rank with LocalExchange).  The
    exchange buffers hold `cap` slots per rank; each phase uses n of them."""
    for r in ranks:
        r.begin()
    rounds = 0
    while True:
        tops = [r.top() for r in ranks]
        n, finished = tops[0]
        if any(t != tops[0] for t in tops):
            raise RuntimeError(f"ranks disagree at the phase top: {tops}")
        if finished:
            break
        assert n <= cap
        for r in ranks:
            r.scan(cand_ptr, meta_ptr, n, False)
        exchange.gather(n, *gather_args)
        parked = [r.da(cand_ptr, meta_ptr, n, False) for r in ranks]
        while parked[0] > 0:
            rounds += 1
            if any(p != parked[0] for p in parked):
                raise RuntimeError(f"ranks disagree on parked chains: {parked}")
            for r in ranks:
                r.scan(cand_ptr, meta_ptr, n, True)
            exchange.gather(n, *gather_args)
            parked = [r.da(cand_ptr, meta_ptr, n, True) for r in ranks]
    return rounds


class ShardedSolver:
    """Prepared sharded solve, reusable across solves of the same instance.

    ``distributed=False``: all ``n_shards`` shards live in this process on
    ``opt.device`` (LocalExchange).  ``distributed=True``: this process is
    rank ``dist.get_rank()`` of ``dist.get_world_size()`` shards on GPU
    LOCAL_RANK (TorchDistExchange over NCCL)."""

    def __init__(self, inst: AssignmentInstance, opt: AssignmentOptions, n_shards: int = 1,
                 K: int = K_DEFAULT, distributed: bool = False, on_the_fly: bool = False):
        _check_options(inst, opt)
        if inst.pts_a is None or inst.pts_b is None:
            raise ParameterError("the sharded path builds slabs from 2-D point sets")
        if distributed:
            import torch.distributed as dist
            rank, world = dist.get_rank(), dist.get_world_size()
            # this rank's GPU: OTPRG_DEVICE, else LOCAL_RANK (one process per GPU)
            device = int(os.environ.get("OTPRG_DEVICE", os.environ.get("LOCAL_RANK", opt.device)))
            self.ranks = [DeviceRank(device)]
            self.ranks[0].prepare(inst, opt.eps, world, rank, K, opt.storage, on_the_fly)
            self.n_shards = world
            self.exchange = TorchDistExchange(rank, world)
        else:
            device = opt.device
            self.ranks = [DeviceRank(device) for _ in range(n_shards)]
            for g, r in enumerate(self.ranks):
                r.prepare(inst, opt.eps, n_shards, g, K, opt.storage, on_the_fly)
            self.n_shards = n_shards
            self.exchange = LocalExchange()
        self.cap = self.ranks[0].cap
        self.cand, self.meta = _buffers(self.n_shards, self.cap, K, device)
        self.gather_args = (self.cand, self.meta, K) if distributed else ()
        # one stream for every context of this process and the exchange:
        # scan -> all-gather -> DA are ordered on it without host syncs
        import torch
        self.stream = torch.cuda.Stream(device=device)
        for r in self.ranks:
            r.set_stream(self.stream.cuda_stream)

    def solve(self, keep_state: bool = False):
        """One full solve (state re-initialised).  Returns (Matching,
        SolveStats) of the first local rank after checking local ranks agree.
        ``keep_state``: also return the state before completion (rank 0's
        snapshot) as a third element, for verify_feasibility."""
        import torch
        with torch.cuda.stream(self.stream):
            rounds = run_phases(self.ranks, self.exchange, self.cand.data_ptr(),
                                self.meta.data_ptr(), self.cap, self.gather_args)
        pre = self.ranks[0].snapshot() if keep_state else None
        outs = [r.finish() for r in self.ranks]
        m0, s0 = outs[0]
        for m, s in outs[1:]:
            if not (np.array_equal(m.match_of_a, m0.match_of_a)
                    and np.array_equal(s.duals_final.y_a, s0.duals_final.y_a)
                    and np.array_equal(s.duals_final.y_b, s0.duals_final.y_b)):
                raise RuntimeError("shards ended in different states")
        s0.device["refill_rounds"] = rounds
        s0.device["n_shards"] = self.n_shards
        return (m0, s0, pre) if keep_state else (m0, s0)

    def timer_start(self):
        for r in self.ranks:
            r.solver.timer_start()

    def timer_stop(self) -> float:
        return max(r.solver.timer_stop() for r in self.ranks)

    def close(self):
        for r in self.ranks:
            r.close()


def solve_assignment_sharded(inst: AssignmentInstance, opt: AssignmentOptions, n_shards: int,
                             K: int = K_DEFAULT, on_the_fly: bool = False):
    """All shards in this process on opt.device (LocalExchange): G logical
    shards on one GPU.  ``on_the_fly``: no kT slabs, costs from the points in
    the scans (OTPRG_FLAG_ON_THE_FLY).  Returns (Matching, SolveStats)."""
    sv = ShardedSolver(inst, opt, n_shards, K, on_the_fly=on_the_fly)
    try:
        return sv.solve()
    finally:
        sv.close()


def solve_assignment_distributed(inst: AssignmentInstance, opt: AssignmentOptions,
                                 K: int = K_DEFAULT, on_the_fly: bool = False):
    """One rank per process/GPU under torch.distributed (NCCL): each process
    calls this with the same instance; every rank returns the same result."""
    sv = ShardedSolver(inst, opt, K=K, distributed=True, on_the_fly=on_the_fly)
    try:
        return sv.solve()
    finally:
        sv.close()
