"""Randomised parity sweep on the device path against the C restatement of
the reference (oracle/): shapes 1..700 per side (both orientations), eps from
0.004 to 0.6 (u8 and u16 storage), dense random / geometric / tied / exact-
multiple costs, a few larger instances that reach the bulk list build and the
team modes.  Every result must be bit-identical (matching, duals, phases,
free_counts, cost)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")


def _instance(rng, kind, n_a, n_b, eps):
    if kind == "random":
        return rng.random((n_a, n_b))
    if kind == "points":
        pa, pb = rng.random((n_a, 2)), rng.random((n_b, 2))
        return otprg.points_cost(pa, pb)
    if kind == "ties":
        return rng.integers(0, 4, (n_a, n_b)) / 4.0
    # exact multiples of eps (scaled_floor boundary cases)
    return np.minimum(rng.integers(0, int(1 / eps) + 1, (n_a, n_b)) * eps, 1.0)


def _check(oracle, cost, eps, storage):
    want = oracle.solve_assignment(cost, eps)
    m, s = otprg.solve_assignment(otprg.AssignmentInstance(*cost.shape, cost),
                                  otprg.AssignmentOptions(eps=eps, storage=storage))
    tag = f"shape={cost.shape} eps={eps} storage={storage}"
    assert np.array_equal(m.match_of_a, want.match_of_a), tag
    assert np.array_equal(s.duals_final.y_a, want.y_a), tag
    assert np.array_equal(s.duals_final.y_b, want.y_b), tag
    assert np.array_equal(s.free_counts, want.free_counts), tag
    assert s.device["cost"] == want.cost, tag


def test_random_sweep_small(oracle):
    rng = np.random.default_rng(20261018)
    kinds = ["random", "points", "ties", "multiples"]
    for trial in range(500):
        n_a = int(rng.integers(1, 700))
        n_b = int(rng.integers(1, 700))
        eps = float(np.exp(rng.uniform(np.log(0.004), np.log(0.6))))
        storage = "u8" if (np.ceil(1 / eps) + 2 <= 253 and trial % 2) else "u16"
        cost = _instance(rng, kinds[trial % 4], n_a, n_b, eps)
        _check(oracle, cost, eps, storage)


def test_random_sweep_larger(oracle):
    """Sizes that take the bulk list build (n_i >= total warps) and 8-warp teams."""
    rng = np.random.default_rng(7)
    for n_a, n_b, eps in ((3000, 2900, 0.02), (2600, 3100, 0.03), (4000, 4000, 0.05)):
        pa, pb = rng.random((n_a, 2)), rng.random((n_b, 2))
        _check(oracle, otprg.points_cost(pa, pb), eps, "u16")
