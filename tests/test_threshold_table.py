"""SURVEY F6 on the CPU: the exact threshold table of the 2-D point cost
(otprg_points_threshold_table) reproduces the oracle's rounded costs
k = scaled_floor(sqrt(dx*dx + dy*dy) / sqrt(2), eps) for every pair, without
sqrt or division (instances.cpp:70-75, core.cpp:26-32)."""
import numpy as np
import pytest

import paper_2203_03732_b200 as otprg
from paper_2203_03732_b200.api import points_threshold_table


def _k_table(pa, pb, thr):
    dx = pa[:, None, 0] - pb[None, :, 0]
    dy = pa[:, None, 1] - pb[None, :, 1]
    d2 = dx * dx + dy * dy  # RN products and sum, no FMA (numpy)
    return np.searchsorted(thr, d2, side="right") - 1


@pytest.mark.parametrize("eps", [0.1, 0.01, 1.0 / 300.0, 0.125, 0.02, 0.003, 0.37])
def test_table_matches_oracle_rounding(oracle, eps):
    thr = points_threshold_table(eps)
    uf = oracle.scaled_floor(1.0, eps)
    assert len(thr) == uf + 2 and thr[0] == 0.0 and np.isinf(thr[-1])
    assert np.all(np.diff(thr[np.isfinite(thr)]) > 0)
    for seed in (1, 2):
        ax, ay, bx, by = oracle.uniform_square_points(700, seed)
        pa, pb = np.stack([ax, ay], 1), np.stack([bx, by], 1)
        want, _, _ = oracle.scale_round_costs(oracle.gen_uniform_square(700, seed), eps)
        np.testing.assert_array_equal(_k_table(pa, pb, thr), want)
    rng = np.random.default_rng(3)  # adversarial: points on a fine grid (many exact ties)
    g = rng.integers(0, 64, (300, 2)) / 64.0
    h = rng.integers(0, 64, (300, 2)) / 64.0
    want, _, _ = oracle.scale_round_costs(otprg.points_cost(g, h), eps)
    np.testing.assert_array_equal(_k_table(g, h, thr), want)


def test_table_rejects_bad_eps():
    with pytest.raises(otprg.ParameterError):
        points_threshold_table(0.0)
