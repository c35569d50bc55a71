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

Drivers: ``resident=True`` (default) runs every round on the device — one
CUDA graph per GPU with a conditional WHILE node (otprg_shard_solve_resident):
the shards of this process on one GPU run in stream order, and shards on other
GPUs (other processes: CUDA IPC handles exchanged over torch.distributed) get
the candidate slots pushed into their exchange blocks over NVLink peer memory
with epoch flags; one host sync per solve.  ``resident=False`` is the
host-driven protocol (one host sync per round): ``DeviceRank`` drives one
otprg_ctx through the C ABI and the exchange is ``LocalExchange`` (all ranks
of the process share one buffer) or ``TorchDistExchange`` (torch.distributed
all_gather: NCCL, or gloo when several ranks share one GPU — the resident
loop's cross-process flag waits need distinct GPUs).
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

    def ipc_export(self, n_groups: int, my_group: int) -> bytes:
        from . import _native as N
        h = (C.c_char * N.IPC_HANDLE_BYTES)()
        self._ok(self._L.otprg_shard_ipc_export(self._ctx, n_groups, my_group, h))
        return bytes(h)

    def ipc_attach(self, handles: list, group_shard_lo: list):
        blob = b"".join(handles)
        lo = np.asarray(group_shard_lo, np.int32)
        self._ok(self._L.otprg_shard_ipc_attach(self._ctx, blob, len(handles), lo.ctypes.data))

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


def solve_resident(ranks):
    """otprg_shard_solve_resident over this process's ranks: (Matching, SolveStats)."""
    L = ranks[0]._L
    n_a, n_b, eps = ranks[0].shape
    r, bufs = ranks[0].solver._result(n_a, n_b, eps)
    arr = (C.c_void_p * len(ranks))(*[x._ctx for x in ranks])
    st = L.otprg_shard_solve_resident(arr, len(ranks), C.byref(r))
    if st:
        ranks[0].solver._raise(st)
    return Solver._pack(r, bufs)


class ShardedSolver:
    """Prepared sharded solve, reusable across solves of the same instance.

    ``distributed=False``: all ``n_shards`` shards live in this process on
    ``opt.device`` (logical shards; ``devices``: one device per shard).
    ``distributed=True``: this process is rank ``dist.get_rank()`` of
    ``dist.get_world_size()`` shards on GPU LOCAL_RANK (or OTPRG_DEVICE).
    ``resident``: device-resident loop (default; across processes it needs
    distinct GPUs per rank), else the host-driven protocol."""

    def __init__(self, inst: AssignmentInstance, opt: AssignmentOptions, n_shards: int = 1,
                 K: int = K_DEFAULT, distributed: bool = False, on_the_fly: bool = False,
                 resident: bool | None = None, devices: list | None = None):
        _check_options(inst, opt)
        if (inst.pts_a is None or inst.pts_b is None) and (inst.img_a is None or inst.img_b is None):
            raise ParameterError("the sharded path builds slabs from 2-D point sets or L1 images")
        self.distributed = distributed
        if distributed:
            import torch.distributed as dist
            rank, world = dist.get_rank(), dist.get_world_size()
            # this rank's GPU: OTPRG_DEVICE, else LOCAL_RANK (one process per GPU)
            device = int(os.environ.get("OTPRG_DEVICE", os.environ.get("LOCAL_RANK", opt.device)))
            self.ranks = [DeviceRank(device)]
            self.ranks[0].prepare(inst, opt.eps, world, rank, K, opt.storage, on_the_fly)
            self.n_shards = world
            self.exchange = TorchDistExchange(rank, world)
            if resident is None:  # the flag waits need one GPU per rank
                import torch
                devs = [None] * world
                dist.all_gather_object(devs, (socket_host(), device))
                resident = len(set(devs)) == world
            if resident:
                ok = 1
                try:
                    h = self.ranks[0].ipc_export(world, rank)
                except Exception:  # noqa: BLE001
                    h, ok = b"", 0
                handles = [None] * world
                dist.all_gather_object(handles, h)
                try:
                    if ok and all(handles):
                        self.ranks[0].ipc_attach(handles, list(range(world)))
                    else:
                        ok = 0
                except Exception:  # noqa: BLE001
                    ok = 0
                oks = [None] * world
                dist.all_gather_object(oks, ok)
                if not all(oks):  # no peer mapping on some rank: the host-driven protocol everywhere
                    resident = False
                    self.resident_error = "CUDA IPC attach failed on some rank"
                    self.ranks[0].prepare(inst, opt.eps, world, rank, K, opt.storage, on_the_fly)
        else:
            devs = list(devices) if devices is not None else [opt.device] * n_shards
            if len(devs) != n_shards:
                raise ParameterError("one device per shard")
            device = devs[0]
            self.ranks = [DeviceRank(d) for d in devs]
            for g, r in enumerate(self.ranks):
                r.prepare(inst, opt.eps, n_shards, g, K, opt.storage, on_the_fly)
            self.n_shards = n_shards
            self.exchange = LocalExchange()
            if resident is None:
                resident = True
            if not resident and len(set(devs)) > 1:
                raise ParameterError("the host-driven protocol keeps in-process shards on one device")
        self.resident = bool(resident)
        self.cap = self.ranks[0].cap
        if not self.resident:
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
        ``keep_state`` (host-driven mode): also return the state before
        completion (rank 0's snapshot) as a third element, for
        verify_feasibility."""
        if self.resident:
            if keep_state:
                raise ParameterError("keep_state needs the host-driven protocol (resident=False)")
            if self.distributed:
                import torch.distributed as dist
                dist.barrier()  # every rank's graph launches after every rank attached
            return solve_resident(self.ranks)
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


def socket_host() -> str:
    import socket
    return socket.gethostname()


def solve_assignment_sharded(inst: AssignmentInstance, opt: AssignmentOptions, n_shards: int,
                             K: int = K_DEFAULT, on_the_fly: bool = False, resident: bool = True,
                             devices: list | None = None):
    """All shards in this process (on opt.device, or one per entry of
    ``devices``).  ``on_the_fly``: no kT slabs, costs from the points in the
    scans (OTPRG_FLAG_ON_THE_FLY).  Returns (Matching, SolveStats)."""
    sv = ShardedSolver(inst, opt, n_shards, K, on_the_fly=on_the_fly, resident=resident, devices=devices)
    try:
        return sv.solve()
    finally:
        sv.close()


def solve_assignment_distributed(inst: AssignmentInstance, opt: AssignmentOptions,
                                 K: int = K_DEFAULT, on_the_fly: bool = False,
                                 resident: bool | None = None):
    """One rank per process/GPU under torch.distributed: each process calls
    this with the same instance; every rank returns the same result."""
    sv = ShardedSolver(inst, opt, K=K, distributed=True, on_the_fly=on_the_fly, resident=resident)
    try:
        return sv.solve()
    finally:
        sv.close()


class MultiSolver:
    """A multi-device context (otprg_create_multi): point instances are
    A-row-sharded over ``devices`` (one shard per entry; a device listed
    several times holds several logical shards) and solved by the resident
    loop; other instances run on the first device.  The C++ drop-in's
    otprg::AssignmentOptions::devices takes the same path."""

    def __init__(self, devices: list, K: int = K_DEFAULT):
        from . import _native as N
        self._L = N.lib()
        self._ctx = C.c_void_p()
        arr = (C.c_int32 * len(devices))(*devices)
        st = self._L.otprg_create_multi(arr, len(devices), C.byref(self._ctx))
        if st:
            from .api import DeviceError
            raise DeviceError(f"otprg_create_multi({devices}) failed with status {st}")
        self.devices = list(devices)
        self._keep = ()
        st = self._L.otprg_set_shard_k(self._ctx, K)
        if st:
            self._raise(st)

    # the Solver helpers work on any object with _L / _ctx / _keep
    _raise = Solver._raise
    _problem = Solver._problem
    _result = Solver._result

    def prepare(self, inst: AssignmentInstance, eps: float, storage: str = "auto", on_the_fly: bool = False):
        from . import _native as N
        p = self._problem(inst, eps, storage)
        if on_the_fly:
            p.flags |= N.FLAG_ON_THE_FLY
        r = N.Result()
        st = self._L.otprg_prepare(self._ctx, C.byref(p), C.byref(r))
        if st:
            self._raise(st)
        self._shape = (inst.n_a, inst.n_b, eps)

    def solve_prepared(self):
        n_a, n_b, eps = self._shape
        r, bufs = self._result(n_a, n_b, eps)
        st = self._L.otprg_solve_prepared(self._ctx, C.byref(r))
        if st:
            self._raise(st)
        return Solver._pack(r, bufs)

    def solve(self, inst: AssignmentInstance, opt: AssignmentOptions, on_the_fly: bool = False):
        self.prepare(inst, opt.eps, opt.storage, on_the_fly)
        return self.solve_prepared()

    def close(self):
        if self._ctx:
            self._L.otprg_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
