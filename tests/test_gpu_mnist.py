"""Config 3 on the GPU: MNIST-shaped L1 costs (load_mnist_pair,
instances.cpp:80-144) — device L1/2 cost + rounding and the full solve,
bit-exact against the unmodified reference (tests/golden/mnist_pins.json).
"""
import json
import os

import numpy as np
import pytest

from golden_util import PIN_KEYS, pins_of

pytestmark = pytest.mark.gpu
otprg = pytest.importorskip("paper_2203_03732_b200")
from paper_2203_03732_b200.instances import make_synthetic_mnist  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mnist_pins.json")


@pytest.fixture(scope="module")
def idx3(tmp_path_factory):
    return make_synthetic_mnist(str(tmp_path_factory.mktemp("mnist") / "synth-idx3"), 20000, 0)


@pytest.fixture(scope="module")
def pins():
    with open(GOLDEN) as f:
        return json.load(f)


def test_l1_rounding_matches_host_formula(idx3, oracle):
    inst = otprg.load_mnist_pair(idx3, 300, 5)
    dense = otprg.l1_cost(inst.img_a, inst.img_b)
    for eps in (0.1, 0.01, 1.0 / 300.0):
        want, uf, uc = oracle.scale_round_costs(dense, eps)
        got = otprg.scale_round_costs(inst, eps)
        np.testing.assert_array_equal(got.k, want)


def test_mnist_solves_match_reference(idx3, pins):
    keys = sorted(k for k, v in pins.items() if v["n_a"] <= 2000)
    assert keys
    loaded = {}
    for key in keys:
        w = pins[key]
        ck = (w["n_a"], w["seed"])
        if ck not in loaded:
            loaded[ck] = otprg.load_mnist_pair(idx3, w["n_a"], w["seed"])
        m, s = otprg.solve_assignment(loaded[ck], otprg.AssignmentOptions(eps=w["eps"]))
        got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts,
                      s.phases, s.sum_ni, s.device["cost"])
        assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}, key


def test_mnist_config3_n10k_eps_sweep(idx3, pins):
    keys = sorted(k for k, v in pins.items() if v["n_a"] == 10000)
    if not keys:
        pytest.skip("n=10k fixtures not generated")
    inst = otprg.load_mnist_pair(idx3, 10000, 1)
    for key in keys:
        w = pins[key]
        m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"]))
        got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts,
                      s.phases, s.sum_ni, s.device["cost"])
        assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}, key


@pytest.mark.parametrize("costs,G,K", [("on_the_fly", 1, 16), ("on_the_fly", 3, 4), ("matrix", 2, 16)])
def test_mnist_sharded_and_on_the_fly(idx3, pins, costs, G, K):
    """North star (1) for d-dim vectors: no rounded matrix at all — the scans
    sum the 784 pixel differences per entry themselves (the reference's
    arithmetic, ascending p, no FMA) — and L1 slabs sharded over G logical
    shards; both bit-exact with the reference pins (n <= 2000 here)."""
    from paper_2203_03732_b200 import sharded
    keys = sorted(k for k, v in pins.items() if v["n_a"] <= 2000)
    loaded = {}
    for key in keys:
        w = pins[key]
        ck = (w["n_a"], w["seed"])
        if ck not in loaded:
            loaded[ck] = otprg.load_mnist_pair(idx3, w["n_a"], w["seed"])
        m, s = sharded.solve_assignment_sharded(loaded[ck], otprg.AssignmentOptions(eps=w["eps"]), G, K=K,
                                                on_the_fly=costs == "on_the_fly")
        got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts,
                      s.phases, s.sum_ni, s.device["cost"])
        assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}, (key, costs, G)


@pytest.mark.slow
def test_mnist_config3_n10k_on_the_fly(idx3, pins):
    """Config 3 at n = 10k with costs on the fly (public API, costs =
    "on_the_fly"): every eps of the sweep bit-exact with the reference."""
    keys = sorted(k for k, v in pins.items() if v["n_a"] == 10000)
    if not keys:
        pytest.skip("n=10k fixtures not generated")
    inst = otprg.load_mnist_pair(idx3, 10000, 1)
    for key in keys:
        w = pins[key]
        m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"], costs="on_the_fly"))
        got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts,
                      s.phases, s.sum_ni, s.device["cost"])
        assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}, key
