"""GPU parity of the A-row-sharded path: G logical shards on
one device (each with its own context, slab and replicated state, exchanging
candidate slots through one shared buffer) must give the reference's result
bit for bit for every G and K, and the torch.distributed (NCCL) driver must
agree with it."""
import os
import socket

import numpy as np
import pytest

from golden_util import PIN_KEYS, pins_of

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")
from paper_2203_03732_b200 import sharded  # noqa: E402


def _pins(m, s):
    return pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                   s.sum_ni, s.device["cost"])


def _check_golden(golden, key, m, s):
    want = golden[key]
    got = _pins(m, s)
    assert {k: got[k] for k in PIN_KEYS} == {k: want[k] for k in PIN_KEYS}, key
    assert bool(s.full_match_termination) == bool(want["full_match_termination"])


@pytest.mark.parametrize("key,G", [
    ("square_n4000_eps0.01_s1", 1), ("square_n4000_eps0.01_s1", 2),
    ("square_n4000_eps0.01_s1", 4), ("square_n4000_eps0.01_s1", 7),
    ("square_n10000_eps0.01_s1", 2), ("square_n10000_eps0.01_s2", 4),
    ("square_n10000_eps0.01_s3", 8), ("square_n3000_eps0.02_s1", 3),
    ("square_n10000_eps0.1_s1", 8), ("square_n1000_eps0.01_s1", 2),
])
def test_sharded_matches_golden(golden, key, G):
    v = golden[key]
    inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
    m, s = sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=v["eps"]), G)
    _check_golden(golden, key, m, s)


@pytest.mark.parametrize("K,G", [(1, 4), (2, 8), (5, 3)])
def test_sharded_forced_rescans(golden, K, G):
    key = "square_n4000_eps0.01_s1"
    v = golden[key]
    inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
    m, s = sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=v["eps"]), G, K=K)
    if K <= 2:
        assert s.device["refill_rounds"] > 0  # truncated lists really forced rescans
    _check_golden(golden, key, m, s)


@pytest.mark.parametrize("storage", ["u8", "u16", "u32"])
def test_sharded_storage(golden, storage):
    key = "square_n2000_eps0.01_s3"
    v = golden[key]
    inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
    m, s = sharded.solve_assignment_sharded(
        inst, otprg.AssignmentOptions(eps=v["eps"], storage=storage), 3)
    _check_golden(golden, key, m, s)


def test_sharded_rectangular_vs_single():
    rng = np.random.default_rng(5)
    for n_a, n_b in ((3000, 1700), (1500, 2600)):
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)),
                                        pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=0.02)
        m1, s1 = otprg.solve_assignment(inst, opt)
        m2, s2 = sharded.solve_assignment_sharded(inst, opt, 3, K=4)
        assert np.array_equal(m1.match_of_a, m2.match_of_a)
        assert np.array_equal(m1.match_of_b, m2.match_of_b)
        assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
        assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
        assert np.array_equal(s1.free_counts, s2.free_counts)
        assert s1.device["cost"] == s2.device["cost"]
        assert s1.swapped == s2.swapped


@pytest.mark.slow
def test_sharded_100k_vs_single():
    inst = otprg.gen_uniform_square(100_000, 1)
    opt = otprg.AssignmentOptions(eps=0.01)
    m1, s1 = otprg.solve_assignment(inst, opt)
    m2, s2 = sharded.solve_assignment_sharded(inst, opt, 8)
    assert np.array_equal(m1.match_of_a, m2.match_of_a)
    assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
    assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
    assert s1.phases == s2.phases and s1.sum_ni == s2.sum_ni


def test_distributed_world1_nccl(golden):
    import torch.distributed as dist
    key = "square_n4000_eps0.01_s1"
    v = golden[key]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("LOCAL_RANK", "0")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
        m, st = sharded.solve_assignment_distributed(inst, otprg.AssignmentOptions(eps=v["eps"]))
        _check_golden(golden, key, m, st)
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_gloo():
    """The multi-process protocol end to end on real kernels: two
    torch.distributed ranks (gloo exchange, both contexts on cuda:0) — golden
    pins and bit-identity with the fused solver at n = 100k
    (scripts/dist_on_one_gpu.py)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, OTPRG_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        "scripts/dist_on_one_gpu.py"], cwd=root, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "DIST OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


# ---- on-the-fly costs (OTPRG_FLAG_ON_THE_FLY) ----

@pytest.mark.parametrize("key,G,K", [
    ("square_n10000_eps0.01_s1", 1, 16), ("square_n10000_eps0.01_s2", 3, 16),
    ("square_n4000_eps0.01_s1", 2, 1), ("square_n10000_eps0.1_s1", 4, 4),
    ("square_n3000_eps0.02_s1", 5, 2), ("square_n1000_eps0.01_s1", 1, 16),
])
def test_on_the_fly_matches_golden(golden, key, G, K):
    """No kT slab: the scans round the 2-D point costs themselves through the
    exact threshold table; results equal the reference's bit for bit."""
    v = golden[key]
    m, s = sharded.solve_assignment_sharded(otprg.gen_uniform_square(v["n_a"], v["seed"]),
                                            otprg.AssignmentOptions(eps=v["eps"]), G, K=K, on_the_fly=True)
    _check_golden(golden, key, m, s)


@pytest.mark.parametrize("storage", ["u8", "u16", "u32"])
def test_on_the_fly_rectangular_and_storage(storage):
    rng = np.random.default_rng(17)
    for n_a, n_b, eps in ((2500, 1300, 0.02), (900, 2100, 0.05), (64, 64, 0.003)):
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)), pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=eps, storage=storage)
        try:
            m1, s1 = otprg.solve_assignment(inst, opt)
        except otprg.ParameterError:
            continue  # storage too narrow for eps
        m2, s2 = sharded.solve_assignment_sharded(inst, opt, 3, K=4, on_the_fly=True)
        assert np.array_equal(m1.match_of_a, m2.match_of_a)
        assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
        assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
        assert np.array_equal(s1.free_counts, s2.free_counts)
        assert s1.device["cost"] == s2.device["cost"] and s1.swapped == s2.swapped


def test_on_the_fly_rejects_tiny_eps():
    inst = otprg.gen_uniform_square(50, 1)
    with pytest.raises(otprg.ParameterError):
        sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=1e-4), 1, on_the_fly=True)


@pytest.mark.parametrize("otf", [False, True])
def test_tiny_instances_with_empty_shards(otf):
    """n below the 512-element shard granularity (all but the last shard
    empty) and below the compaction's 148 blocks, many times over."""
    rng = np.random.default_rng(23)
    for trial in range(40):
        n_a, n_b = int(rng.integers(1, 150)), int(rng.integers(1, 150))
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)), pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=float(rng.choice([0.01, 0.05, 0.2])))
        m1, s1 = otprg.solve_assignment(inst, opt)
        m2, s2 = sharded.solve_assignment_sharded(inst, opt, int(rng.integers(1, 5)), K=int(rng.choice([1, 16])),
                                                  on_the_fly=otf)
        assert np.array_equal(m1.match_of_a, m2.match_of_a), trial
        assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b), trial
        assert s1.phases == s2.phases, trial


@pytest.mark.parametrize("shift,scale", [(0.0, 1.0), (1000.0, 1.0), (-3.5e4, 0.7), (0.25, 1e-3)])
def test_on_the_fly_shifted_scaled_points(shift, scale):
    """The on-the-fly scans test thr[m] <= d2 < thr[m+1] on the double
    points (branch-free, out-of-range lanes masked).  Shifted / scaled point
    sets (costs still in [0, 1]) must give the dense solver's result bit for
    bit."""
    rng = np.random.default_rng(31)
    n = 3000
    pa = shift + scale * rng.random((n, 2))
    pb = shift + scale * rng.random((n, 2))
    inst = otprg.AssignmentInstance(n, n, pts_a=pa, pts_b=pb)
    opt = otprg.AssignmentOptions(eps=0.01)
    m1, s1 = otprg.solve_assignment(inst, opt)
    m2, s2 = sharded.solve_assignment_sharded(inst, opt, 2, K=16, on_the_fly=True)
    assert np.array_equal(m1.match_of_a, m2.match_of_a)
    assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
    assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
    assert np.array_equal(s1.free_counts, s2.free_counts)
    assert s1.device["cost"] == s2.device["cost"]


@pytest.mark.slow
def test_on_the_fly_100k_vs_single():
    inst = otprg.gen_uniform_square(100_000, 1)
    opt = otprg.AssignmentOptions(eps=0.01)
    m1, s1 = otprg.solve_assignment(inst, opt)
    m2, s2 = sharded.solve_assignment_sharded(inst, opt, 1, on_the_fly=True)
    assert np.array_equal(m1.match_of_a, m2.match_of_a)
    assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
    assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
    assert s1.phases == s2.phases and s1.sum_ni == s2.sum_ni
