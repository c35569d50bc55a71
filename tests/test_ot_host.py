"""CPU tests for the OT host path: instance generator, theta scaling
(scale_and_round, ot.cpp:109-128) and their KATs (test_ot.cpp:62-88),
against the unmodified reference."""
import numpy as np
import pytest

import paper_2203_03732_b200 as otprg


def test_random_ot_rational_matches_reference(reference):
    for n_a, n_b, seed in ((6, 4, 3), (10, 10, 7), (120, 80, 99)):
        inst = otprg.gen_random_ot_rational(n_a, n_b, seed)
        mu, nu, cost = reference.gen_random_ot_rational(n_a, n_b, seed)
        assert inst.mu.tobytes() == mu.tobytes()
        assert inst.nu.tobytes() == nu.tobytes()
        assert inst.cost.tobytes() == cost.tobytes()


def test_scale_and_round_kats():
    # test_ot.cpp:62-72: theta = 16, d = ceil(8.8), ceil(7.2), s = floor(4.8), floor(11.2)
    inst = otprg.OTInstance(np.array([0.55, 0.45]), np.array([0.3, 0.7]), np.array([[0.1, 0.2], [0.3, 0.4]]))
    sm = otprg.scale_and_round(inst, 0.5)
    assert sm.theta == 16.0
    assert list(sm.d) == [9, 8] and list(sm.s) == [4, 11]
    # test_ot.cpp:74-80: exact dyadic multiples unchanged
    inst = otprg.OTInstance(np.array([0.25, 0.75]), np.array([0.5, 0.5]), np.zeros((2, 2)))
    sm = otprg.scale_and_round(inst, 0.5)
    assert list(sm.d) == [4, 12] and list(sm.s) == [8, 8]


def test_scale_and_round_matches_reference(reference):
    for seed in range(1, 11):  # test_ot.cpp:82-88
        inst = otprg.gen_random_ot_rational(6, 4, seed)
        sm = otprg.scale_and_round(inst, 0.23)
        d, s, th = reference.scale_and_round(inst.mu, inst.nu, inst.cost, 0.23)
        assert sm.theta == th and np.array_equal(sm.d, d) and np.array_equal(sm.s, s)
        assert sm.total_s() <= sm.theta + 1e-9 <= sm.total_d() + 2e-9


def test_scale_and_round_errors():
    inst = otprg.OTInstance(np.array([1.0]), np.array([0.9]), np.array([[0.2]]))
    with pytest.raises(otprg.InputError):  # masses must sum to 1 (ot.cpp:78-83)
        otprg.scale_and_round(inst, 0.1)
    inst = otprg.OTInstance(np.array([1.0]), np.array([1.0]), np.array([[0.2]]))
    for eps in (0.0, 1.0):
        with pytest.raises(otprg.ParameterError):
            otprg.scale_and_round(inst, eps)
