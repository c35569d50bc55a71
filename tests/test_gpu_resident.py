"""The device-resident sharded loop: every
round of every phase inside one CUDA graph per device (conditional WHILE
node), one host sync per solve.

* the peer exchange (push + epoch flags) on one GPU, emulated as one
  cooperative grid over all groups (otprg_selftest_exchange);
* resident solves of G logical shards bit-identical to the golden pins and to
  the host-driven protocol, slab and on-the-fly, K = 1 (many refill rounds)
  and 16; repeated solves reuse the graphs; re-prepare invalidates them;
* the multi-device context (otprg_create_multi), the C-ABI entry the C++
  drop-in's AssignmentOptions::devices uses;
* real multi-GPU runs (>= 2 visible GPUs only).
"""
import ctypes as C

import numpy as np
import pytest

from golden_util import PIN_KEYS, pins_of

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")
from paper_2203_03732_b200 import _native as N  # noqa: E402
from paper_2203_03732_b200 import sharded  # noqa: E402


def _pins(m, s):
    return pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                   s.sum_ni, s.device["cost"])


def _check(golden, key, m, s):
    want = golden[key]
    got = _pins(m, s)
    assert {k: got[k] for k in PIN_KEYS} == {k: want[k] for k in PIN_KEYS}, key


@pytest.mark.parametrize("n_groups,spg,ib,K", [(2, 1, 1000, 16), (3, 2, 777, 4), (8, 1, 300, 1),
                                               (2, 3, 1, 32), (5, 1, 4096, 16)])
def test_exchange_selftest(n_groups, spg, ib, K):
    mism = C.c_int64(-1)
    st = N.lib().otprg_selftest_exchange(0, n_groups, spg, ib, K, 4, C.byref(mism))
    assert st == 0 and mism.value == 0


@pytest.mark.parametrize("key,G,K,otf", [
    ("square_n4000_eps0.01_s1", 1, 16, False), ("square_n4000_eps0.01_s1", 4, 1, False),
    ("square_n10000_eps0.01_s2", 8, 16, False), ("square_n10000_eps0.01_s3", 3, 2, False),
    ("square_n10000_eps0.1_s1", 2, 4, False), ("square_n1000_eps0.01_s1", 2, 16, False),
    ("square_n4000_eps0.01_s1", 2, 1, True), ("square_n10000_eps0.01_s1", 1, 16, True),
    ("square_n10000_eps0.1_s1", 4, 4, True), ("square_n3000_eps0.02_s1", 5, 2, True),
])
def test_resident_matches_golden_and_host_driven(golden, key, G, K, otf):
    v = golden[key]
    inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
    opt = otprg.AssignmentOptions(eps=v["eps"])
    sv = sharded.ShardedSolver(inst, opt, G, K=K, on_the_fly=otf, resident=True)
    try:
        m, s = sv.solve()
        _check(golden, key, m, s)
        m2, s2 = sv.solve()  # the cached graphs again
        _check(golden, key, m2, s2)
        assert s2.device["n_shards"] == G
    finally:
        sv.close()
    mh, sh = sharded.solve_assignment_sharded(inst, opt, G, K=K, on_the_fly=otf, resident=False)
    _check(golden, key, mh, sh)
    assert sh.device["refill_rounds"] == s.device["refill_rounds"]


def test_resident_reprepare_and_rectangular():
    rng = np.random.default_rng(8)
    for n_a, n_b in ((3000, 1700), (1500, 2600), (130, 90)):
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)), pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=0.02)
        m1, s1 = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.02, costs="matrix"))
        for otf in (False, True):
            m2, s2 = sharded.solve_assignment_sharded(inst, opt, 3, K=4, on_the_fly=otf)
            assert np.array_equal(m1.match_of_a, m2.match_of_a)
            assert np.array_equal(m1.match_of_b, m2.match_of_b)
            assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
            assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
            assert np.array_equal(s1.free_counts, s2.free_counts)
            assert s1.device["cost"] == s2.device["cost"]


@pytest.mark.parametrize("devices,otf", [([0], False), ([0, 0], False), ([0, 0, 0, 0], True), ([0] * 8, False)])
def test_multi_device_context(golden, devices, otf):
    key = "square_n10000_eps0.01_s1"
    v = golden[key]
    ms = sharded.MultiSolver(devices)
    try:
        for seed in (1, 2, 1):  # re-prepare between instances (plans rebuilt)
            k = f"square_n10000_eps0.01_s{seed}"
            m, s = ms.solve(otprg.gen_uniform_square(v["n_a"], seed), otprg.AssignmentOptions(eps=v["eps"]),
                            on_the_fly=otf)
            _check(golden, k, m, s)
            assert s.device["n_shards"] == len(devices)
        # non-point instances run on the first device
        dense = otprg.AssignmentInstance(300, 300, otprg.points_cost(*[np.random.default_rng(3).random((300, 2))
                                                                       for _ in range(2)]))
        m1, s1 = ms.solve(dense, otprg.AssignmentOptions(eps=0.05))
        m2, s2 = otprg.Solver(0).solve(dense, otprg.AssignmentOptions(eps=0.05))
        assert np.array_equal(m1.match_of_a, m2.match_of_a) and s1.phases == s2.phases
    finally:
        ms.close()


def test_resident_tiny_instances():
    rng = np.random.default_rng(29)
    for trial in range(25):
        n_a, n_b = int(rng.integers(1, 150)), int(rng.integers(1, 150))
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)), pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=float(rng.choice([0.01, 0.05, 0.2])))
        m1, s1 = otprg.solve_assignment(inst, opt)
        m2, s2 = sharded.solve_assignment_sharded(inst, opt, int(rng.integers(1, 5)), K=int(rng.choice([1, 16])),
                                                  on_the_fly=bool(trial % 2))
        assert np.array_equal(m1.match_of_a, m2.match_of_a), trial
        assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b), trial
        assert s1.phases == s2.phases, trial


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("_gpus() < 2")
def test_two_gpus_resident(golden):
    key = "square_n10000_eps0.01_s2"
    v = golden[key]
    inst = otprg.gen_uniform_square(v["n_a"], v["seed"])
    m, s = sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=v["eps"]), 2, devices=[0, 1])
    _check(golden, key, m, s)
