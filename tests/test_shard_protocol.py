"""CPU tests of the A-row-sharded protocol: the numpy model of
the shard kernels (tests/shard_model.py) driven by the product's own
``sharded.run_phases`` loop, locally and over a gloo world_size-2 exchange,
must reproduce the oracle's sequential solve bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from shard_model import NumpyRank  # noqa: E402

from paper_2203_03732_b200.sharded import LocalExchange, TorchDistExchange, run_phases  # noqa: E402


def _kT_square(oracle, n, seed, eps):
    cost = oracle.gen_uniform_square(n, seed)
    k, _, _ = oracle.scale_round_costs(cost, eps)
    return np.ascontiguousarray(k.T)


def _kT_rect(oracle, n_a, n_b, seed, eps):
    rng = np.random.default_rng(seed)
    cost = rng.random((n_a, n_b))
    k, _, _ = oracle.scale_round_costs(cost, eps)
    return np.ascontiguousarray(k.T)  # (n_b, n_a), n_a >= n_b


def _run_local(kT, eps, G, K, align):
    ranks = [NumpyRank(align) for _ in range(G)]
    for g, r in enumerate(ranks):
        r.prepare(kT, eps, G, g, K)
    cap = kT.shape[0]
    cand = np.full(G * cap * K, -1, np.int32)
    meta = np.zeros(G * cap * 2, np.int32)
    rounds = run_phases(ranks, LocalExchange(), cand, meta, cap)
    outs = [r.finish() for r in ranks]
    for o in outs[1:]:
        for key in ("match_of_a", "y_a", "y_b", "free_counts"):
            assert np.array_equal(o[key], outs[0][key])
    return outs[0], rounds


def _check(out, ref):
    assert out["phases"] == ref.phases
    assert out["sum_ni"] == ref.sum_ni
    assert np.array_equal(out["free_counts"], ref.free_counts)
    assert np.array_equal(out["match_of_a"], ref.match_of_a)
    assert np.array_equal(out["match_of_b"], ref.match_of_b)
    assert np.array_equal(out["y_a"], ref.y_a)
    assert np.array_equal(out["y_b"], ref.y_b)


@pytest.mark.parametrize("G,K,align", [(1, 16, 16), (2, 16, 16), (3, 4, 16), (4, 1, 8), (4, 2, 32)])
def test_local_square(oracle, G, K, align):
    eps = 0.1
    kT = _kT_square(oracle, 256, 1, eps)
    ref = oracle.solve_rounded(kT, eps)
    out, rounds = _run_local(kT, eps, G, K, align)
    _check(out, ref)
    if G > 1 and K == 1:
        assert rounds > 0  # the truncated lists really forced rescans


def test_local_rect(oracle):
    eps = 0.15
    kT = _kT_rect(oracle, 300, 170, 7, eps)
    ref = oracle.solve_rounded(kT, eps)
    for G, K in ((2, 3), (5, 2)):
        out, _ = _run_local(kT, eps, G, K, 16)
        _check(out, ref)


def _worker(rank, world, port, kT, eps, K, align, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        r = NumpyRank(align)
        r.prepare(kT, eps, world, rank, K)
        cap = kT.shape[0]
        cand = torch.full((world * cap * K,), -1, dtype=torch.int32)
        meta = torch.zeros((world * cap * 2,), dtype=torch.int32)
        rounds = run_phases([r], TorchDistExchange(rank, world), cand.numpy(), meta.numpy(), cap,
                            (cand, meta, K))
        out = r.finish()
        q.put((rank, rounds, {k: np.asarray(v) for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2(oracle):
    eps, K, align = 0.1, 2, 16
    kT = _kT_square(oracle, 200, 3, eps)
    ref = oracle.solve_rounded(kT, eps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kT, eps, K, align, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    assert res[0][1] == res[1][1]
    for _, _, out in res:
        out["phases"], out["sum_ni"] = int(out["phases"]), int(out["sum_ni"])
        _check(out, ref)
