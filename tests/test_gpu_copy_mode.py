"""Copy mode on the device (AssignmentOptions::demand_groups /
supply_groups, assignment.cpp:81-103 scan order and :241-250 supply lift)
against the UNMODIFIED reference on materialised copy instances built like the
reference's tests (test_ot.cpp:40-58 materialize, :234-346).  Bit-exact."""
import numpy as np
import pytest

from golden_util import random_instance

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")


def materialize(orig_cost, d_copies, s_copies):
    dg = np.repeat(np.arange(len(d_copies)), d_copies).astype(np.int32)
    sg = np.repeat(np.arange(len(s_copies)), s_copies).astype(np.int32)
    return orig_cost[np.ix_(dg, sg)], dg, sg


def _cases(seed, trials, max_vertices, max_copies, eps_choices):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < trials:
        n_a = int(rng.integers(1, max_vertices + 1))
        n_b = int(rng.integers(1, max_vertices + 1))
        orig = random_instance(n_a, n_b, int(rng.integers(1, 1 << 30)))
        d = rng.integers(1, max_copies + 1, n_a)
        s, total_s = [], 0
        for _ in range(n_b):
            room = int(d.sum()) - total_s
            c = int(rng.integers(0, room + 1)) if room > 0 else 0
            s.append(c)
            total_s += c
        if total_s == 0:
            continue
        out.append((orig, d, np.array(s), float(rng.choice(eps_choices))))
    return out


def _compare(reference, cost, dg, sg, eps, check):
    want = reference.solve_assignment_groups(cost, eps, dg, sg, check_invariants=check)
    m, s = otprg.solve_assignment(otprg.AssignmentInstance(*cost.shape, cost),
                                  otprg.AssignmentOptions(eps=eps, demand_groups=dg, supply_groups=sg,
                                                          check_invariants=check))
    np.testing.assert_array_equal(m.match_of_a, want.match_of_a)
    np.testing.assert_array_equal(m.match_of_b, want.match_of_b)
    np.testing.assert_array_equal(s.duals_final.y_a, want.y_a)
    np.testing.assert_array_equal(s.duals_final.y_b, want.y_b)
    np.testing.assert_array_equal(s.free_counts, want.free_counts)
    assert s.phases == want.phases and s.sum_ni == want.sum_ni
    assert s.device["cost"] == want.cost
    assert bool(s.full_match_termination) == bool(want.full_match_termination)


def test_copy_mode_micro_grid(reference):
    """test_ot.cpp:234-290: up to 3 x 3 originals, 1-3 copies, eps 0.2-0.5."""
    for orig, d, s, eps in _cases(2024, 40, 3, 3, [0.2, 0.3, 0.4, 0.5]):
        cost, dg, sg = materialize(orig, d, s)
        _compare(reference, cost, dg, sg, eps, check=True)


def test_copy_mode_larger(reference):
    """test_ot.cpp:292-330: 2-5 originals with up to 12 copies each."""
    for orig, d, s, eps in _cases(777, 25, 5, 12, [0.1, 0.15, 0.2, 0.25, 0.3]):
        cost, dg, sg = materialize(orig, d, s)
        _compare(reference, cost, dg, sg, eps, check=True)


def test_copy_mode_at_scale(reference):
    """Hundreds of copies of 40 x 30 originals (materialised ~1000 x ~700)."""
    rng = np.random.default_rng(5)
    orig = random_instance(40, 30, 99)
    d = rng.integers(10, 40, 40)
    s = rng.integers(5, 30, 30)
    while s.sum() > d.sum():
        s[np.argmax(s)] -= 1
    cost, dg, sg = materialize(orig, d, s)
    for eps in (0.05, 0.02):
        _compare(reference, cost, dg, sg, eps, check=False)


def test_copy_mode_observer_runs():
    orig = random_instance(4, 3, 11)
    cost, dg, sg = materialize(orig, np.array([3, 2, 4, 1]), np.array([2, 3, 4]))
    seen = []

    def obs(snap):
        # E' lists come in the grouped scan order: demand group ascending
        for lst in snap.workset.e_admissible:
            assert list(dg[lst]) == sorted(dg[lst])
        seen.append(snap.phase)

    m, s = otprg.solve_assignment(otprg.AssignmentInstance(*cost.shape, cost),
                                  otprg.AssignmentOptions(eps=0.2, demand_groups=dg, supply_groups=sg,
                                                          observer=obs, check_invariants=True))
    assert seen == list(range(1, s.phases + 1))
