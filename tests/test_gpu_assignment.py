"""GPU parity tests: the CUDA path through the C ABI vs the reference.

Every case compares the full result — matching, integer duals (internal
orientation), phase count, free_counts, Σn_i, swapped /
full_match_termination flags and the cost bits — with fixtures produced by
the UNMODIFIED reference (tests/golden/make_golden.py -> oracle/_ref) and,
for ad-hoc instances, with the C oracle restatement.  Bar: bit-exact.

Structure mirrors the reference's tests/test_assignment.cpp and
tests/test_core.cpp.
"""
import re

import numpy as np
import pytest

from golden_util import PIN_KEYS, load_arrays, pins_of, random_instance

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")


def _solve(inst, eps, storage="auto"):
    return otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps, storage=storage))


def _pins(m, s):
    return pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                   s.sum_ni, s.device["cost"])


def _assert_matches_golden(key, want, m, s):
    got = _pins(m, s)
    if any(got[k] != want[k] for k in PIN_KEYS):
        arr = load_arrays(key)
        fc = np.asarray(arr["free_counts"], np.int64)
        n = min(len(fc), len(s.free_counts))
        first = int(np.argmax(fc[:n] != s.free_counts[:n])) if (fc[:n] != s.free_counts[:n]).any() else n
        raise AssertionError(
            f"{key}: got {got} want {{{', '.join(f'{k}: {want[k]}' for k in PIN_KEYS)}}}; "
            f"first free_counts divergence at phase {first + 1}; "
            f"match mismatches {(arr['match_of_a'] != m.match_of_a).sum()}")
    assert bool(s.swapped) == bool(want["swapped"])
    assert bool(s.full_match_termination) == bool(want["full_match_termination"])


def _square_cases(golden, max_n):
    return sorted(k for k, v in golden.items() if v["kind"] == "square" and v["n_a"] <= max_n)


# ---- KATs (test_core.cpp:22-37, test_assignment.cpp:163-185) --------------

def _single(c):
    return otprg.AssignmentInstance(1, 1, np.full((1, 1), c))


def test_scale_round_costs_kats():
    assert otprg.scale_round_costs(_single(0.57), 0.1).k[0, 0] == 5
    assert otprg.scale_round_costs(_single(0.0), 0.1).k[0, 0] == 0
    sc = otprg.scale_round_costs(_single(1.0), 0.1)
    assert sc.k[0, 0] == 10 and float(sc.k[0, 0]) * sc.eps == 1.0


@pytest.mark.parametrize("eps", [0.0, 1.0, -0.1, 1e-12])
def test_scale_round_costs_rejects_bad_eps(eps):
    with pytest.raises(otprg.ParameterError):
        otprg.scale_round_costs(_single(0.5), eps)


def test_cost_outside_unit_interval_is_parameter_error():
    inst = otprg.AssignmentInstance(2, 2, np.array([[0.1, 0.2], [0.3, 1.5]]))
    with pytest.raises(otprg.ParameterError):
        otprg.Solver(0).solve(inst, otprg.AssignmentOptions(eps=0.1))


@pytest.mark.parametrize("costs", ["matrix", "on_the_fly"])
def test_point_cost_outside_unit_interval_is_parameter_error(costs):
    """core.cpp:15-21 for point instances: scaled points give
    costs above 1 and must be rejected on both cost paths with the reference's
    message (first offending (a, b) in row-major order), never truncated."""
    inst = otprg.gen_uniform_square(300, 4)
    big = otprg.AssignmentInstance(300, 300, pts_a=inst.pts_a * 2.0, pts_b=inst.pts_b * 2.0)
    want = None
    dense = otprg.points_cost(big.pts_a, big.pts_b)
    bad = np.argwhere(~((dense >= 0.0) & (dense <= 1.0)))[0]
    want = f"cost entry outside [0,1] at ({bad[0]},{bad[1]}): {dense[bad[0], bad[1]]:f}"
    with pytest.raises(otprg.ParameterError, match=re.escape(want)):
        otprg.solve_assignment(big, otprg.AssignmentOptions(eps=0.01, costs=costs))
    nan_a = inst.pts_a.copy()
    nan_a[7, 1] = np.nan
    with pytest.raises(otprg.ParameterError, match=re.escape("at (7,0)")):
        otprg.solve_assignment(otprg.AssignmentInstance(300, 300, pts_a=nan_a, pts_b=inst.pts_b),
                               otprg.AssignmentOptions(eps=0.01, costs=costs))
    # the boundary itself is legal: the corners of the unit square are at cost 1
    corners = otprg.AssignmentInstance(2, 2, pts_a=np.array([[0.0, 0.0], [1.0, 1.0]]),
                                       pts_b=np.array([[1.0, 1.0], [0.0, 0.0]]))
    m, s = otprg.solve_assignment(corners, otprg.AssignmentOptions(eps=0.1, costs=costs))
    assert m.size() == 2


def test_one_by_one_phase_counts():
    m, s = _solve(_single(0.375), 0.125)
    assert m.match_of_a[0] == 0
    assert s.phases == 4
    assert list(s.free_counts) == [1, 1, 1, 1]
    assert s.duals_final.y_b[0] == 4 and s.duals_final.y_a[0] == -1
    assert s.device["cost"] == 0.375
    m2, s2 = _solve(_single(0.3), 0.1)
    assert s2.phases == 3 and s2.duals_final.y_b[0] == 3
    assert s2.device["cost"] == 0.3


def test_coarse_eps_completes_by_index():
    inst = otprg.AssignmentInstance(10, 10, random_instance(10, 10, 2024))
    m, s = _solve(inst, 0.99)
    assert m.size() == 10
    m.validate()


# ---- rounding parity -----------------------------------------------------

@pytest.mark.parametrize("eps", [0.1, 0.01, 1.0 / 300.0, 0.125, 0.07, 0.003])
def test_rounding_dense_and_points_match_oracle(oracle, eps):
    n = 700
    pts = oracle.uniform_square_points(n, 5)
    cost = oracle.gen_uniform_square(n, 5)
    want, uf, uc = oracle.scale_round_costs(cost, eps)
    inst_d = otprg.AssignmentInstance(n, n, cost)
    sc = otprg.scale_round_costs(inst_d, eps)
    assert (sc.unit_floor, sc.unit_ceil) == (uf, uc)
    np.testing.assert_array_equal(sc.k, want)
    inst_p = otprg.AssignmentInstance(n, n, None, np.stack(pts[:2], 1), np.stack(pts[2:], 1))
    np.testing.assert_array_equal(otprg.scale_round_costs(inst_p, eps).k, want)


@pytest.mark.parametrize("eps", [0.01, 0.1, 1.0 / 300.0, 0.125, 0.003, 1.0 / 8000.0, 0.07])
def test_points_rounding_at_level_boundaries(oracle, eps):
    """K2 decides most entries from a float estimate and consults the exact
    threshold table only near a level boundary: points placed a few ulps on
    either side of every level's threshold distance (and random ones) must
    round exactly like the reference's scale_round_costs of the dense cost."""
    from paper_2203_03732_b200 import _native as N
    import ctypes as C
    n = N.lib().otprg_points_threshold_table(eps, None, 0)
    thr = np.zeros(n)
    N.lib().otprg_points_threshold_table(eps, thr.ctypes.data, n)
    rng = np.random.default_rng(int(1 / eps))
    levels = np.arange(1, n - 1)
    if len(levels) > 600:
        levels = np.sort(rng.choice(levels, 600, replace=False))
    pts = []
    for j in levels:
        r0 = np.sqrt(thr[j])
        for d in range(-3, 4):
            r = r0
            for _ in range(abs(d)):
                r = np.nextafter(r, np.inf if d > 0 else -np.inf)
            th = rng.random() * np.pi / 2
            pts.append((r, 0.0))
            pts.append((r * np.cos(th), r * np.sin(th)))
    pts = np.clip(np.array(pts), 0.0, 1.0)
    pb = np.concatenate([pts, rng.random((500, 2))])
    pa = np.array([[0.0, 0.0], [1.0, 1.0], [0.25, 0.75]])
    # shifted copies: float coordinates lose precision far from the origin (wider margin)
    shift = 777.0
    for A, B in ((pa, pb), (pb, pa), (pa + shift, pb + shift)):
        inst = otprg.AssignmentInstance(len(A), len(B), pts_a=A, pts_b=B)
        got = otprg.scale_round_costs(inst, eps).k
        want = oracle.scale_round_costs(otprg.points_cost(A, B), eps)[0]
        assert np.array_equal(got, want), int((got != want).sum())


def test_rounding_unbalanced_both_orientations(oracle):
    for n_a, n_b in ((37, 301), (301, 37)):
        cost = random_instance(n_a, n_b, 99)
        want, _, _ = oracle.scale_round_costs(cost, 0.007)
        for storage in ("u16", "auto"):
            got = otprg.scale_round_costs(otprg.AssignmentInstance(n_a, n_b, cost), 0.007, storage)
            np.testing.assert_array_equal(got.k, want)


# ---- full-solve parity against the reference's own outputs ---------------

def test_random_instances_match_reference(golden):
    keys = sorted(k for k, v in golden.items() if v["kind"] == "random")
    assert keys
    for key in keys:
        w = golden[key]
        inst = otprg.AssignmentInstance(w["n_a"], w["n_b"], random_instance(w["n_a"], w["n_b"], w["seed"]))
        m, s = _solve(inst, w["eps"])
        _assert_matches_golden(key, w, m, s)
        m.validate()


def test_square_points_match_reference(golden):
    for key in _square_cases(golden, 4000):
        w = golden[key]
        inst = otprg.gen_uniform_square(w["n_a"], w["seed"])
        m, s = _solve(inst, w["eps"])
        _assert_matches_golden(key, w, m, s)


def test_square_dense_match_reference(golden):
    for key in _square_cases(golden, 1000)[:12]:
        w = golden[key]
        inst = otprg.gen_uniform_square(w["n_a"], w["seed"], dense=True)
        m, s = _solve(inst, w["eps"])
        _assert_matches_golden(key, w, m, s)


def test_config2_n10k_eps001_seeds_1_2_3(golden):
    for seed in (1, 2, 3):
        key = f"square_n10000_eps0.01_s{seed}"
        w = golden[key]
        inst = otprg.gen_uniform_square(10000, seed)
        for storage in ("u8", "u16", "u32"):
            m, s = _solve(inst, 0.01, storage)
            _assert_matches_golden(key, w, m, s)


def test_config2_dense_f64_input(golden):
    key = "square_n10000_eps0.01_s1"
    inst = otprg.gen_uniform_square(10000, 1, dense=True)
    m, s = _solve(inst, 0.01)
    _assert_matches_golden(key, golden[key], m, s)


def test_large_eps_long_chains(golden):
    for key in ("square_n10000_eps0.1_s1", "square_n10000_eps0.05_s1", "square_n4000_eps0.1_s1"):
        w = golden[key]
        m, s = _solve(otprg.gen_uniform_square(w["n_a"], w["seed"]), w["eps"])
        _assert_matches_golden(key, w, m, s)


def test_storage_widths_agree_and_repeat_is_deterministic():
    inst = otprg.gen_uniform_square(3000, 11)
    solver = otprg.Solver(0)
    solver.prepare(inst, 0.02, "u8")
    m1, s1 = solver.solve_prepared()
    m2, s2 = solver.solve_prepared()
    solver.prepare(inst, 0.02, "u16")
    m3, s3 = solver.solve_prepared()
    solver.prepare(inst, 0.02, "u32")
    m4, s4 = solver.solve_prepared()
    for m, s in ((m2, s2), (m3, s3), (m4, s4)):
        np.testing.assert_array_equal(m.match_of_a, m1.match_of_a)
        np.testing.assert_array_equal(s.duals_final.y_a, s1.duals_final.y_a)
        np.testing.assert_array_equal(s.duals_final.y_b, s1.duals_final.y_b)
        np.testing.assert_array_equal(s.free_counts, s1.free_counts)
    solver.close()


def test_adhoc_unbalanced_vs_oracle(oracle):
    rng = np.random.default_rng(3)
    for n_a, n_b, eps in ((513, 200, 0.02), (200, 513, 0.02), (1, 7, 0.3), (7, 1, 0.3), (64, 64, 0.004)):
        cost = rng.random((n_a, n_b))
        want = oracle.solve_assignment(cost, eps)
        m, s = _solve(otprg.AssignmentInstance(n_a, n_b, cost), eps)
        np.testing.assert_array_equal(m.match_of_a, want.match_of_a)
        np.testing.assert_array_equal(m.match_of_b, want.match_of_b)
        np.testing.assert_array_equal(s.duals_final.y_a, want.y_a)
        np.testing.assert_array_equal(s.duals_final.y_b, want.y_b)
        np.testing.assert_array_equal(s.free_counts, want.free_counts)
        assert s.device["cost"] == want.cost and s.swapped == want.swapped


# ---- unbalanced instances at scale (assignment.cpp:385-399)
def _rect_pins():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "assign_rect_pins.json")
    with open(p) as f:
        return json.load(f)


@pytest.mark.parametrize("key", sorted(_rect_pins()))
@pytest.mark.parametrize("form", ["points", "dense"])
def test_unbalanced_at_scale_match_reference(key, form):
    w = _rect_pins()[key]
    big = otprg.gen_uniform_square(max(w["n_a"], w["n_b"]), w["seed"])
    pa, pb = big.pts_a[: w["n_a"]], big.pts_b[: w["n_b"]]
    if form == "points":
        inst = otprg.AssignmentInstance(w["n_a"], w["n_b"], pts_a=pa, pts_b=pb,
                                        norm_factor=big.norm_factor)
    else:
        inst = otprg.AssignmentInstance(w["n_a"], w["n_b"], otprg.points_cost(pa, pb))
    m, s = _solve(inst, w["eps"])
    got = _pins(m, s)
    assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}, key
    assert bool(s.swapped) == bool(w["swapped"])
    assert m.size() == min(w["n_a"], w["n_b"])


# ---- the phase-1 scan's split rows (propose_kernels.cu) ---------------------
@pytest.mark.parametrize("storage", ["u8", "u16", "u32"])
def test_phase1_split_rows_match_oracle(oracle, storage):
    """Few long rows: the phase-1 scan splits every row over several warps,
    with warps of empty item ranges in between (n_b * chunks < warps), and the
    last arriver of each row merges the pieces.  Repeated solves on one
    context reuse the arrival counters.  Bit-exact vs the C oracle."""
    rng = np.random.default_rng(99)
    sv = otprg.Solver(0)
    try:
        for n_a, n_b, eps in ((30000, 40, 0.05), (12000, 300, 0.02), (9000, 2, 0.1), (30000, 40, 0.05)):
            pa, pb = rng.random((n_a, 2)), rng.random((n_b, 2))
            cost = otprg.points_cost(pa, pb)
            cost[:, 0] = np.where(rng.random(n_a) < 0.002, 0.0, cost[:, 0])  # zeros spread over row 0
            want = oracle.solve_assignment(cost, eps)
            for inst in (otprg.AssignmentInstance(n_a, n_b, cost),
                         otprg.AssignmentInstance(n_b, n_a, np.ascontiguousarray(cost.T))):
                m, s = sv.solve(inst, otprg.AssignmentOptions(eps=eps, storage=storage))
                if inst.n_a == n_a:
                    np.testing.assert_array_equal(m.match_of_a, want.match_of_a)
                    np.testing.assert_array_equal(s.duals_final.y_a, want.y_a)
                    np.testing.assert_array_equal(s.duals_final.y_b, want.y_b)
                    np.testing.assert_array_equal(s.free_counts, want.free_counts)
                    assert s.device["cost"] == want.cost
                else:  # transposed instance: the same internal orientation (swapped)
                    want_t = oracle.solve_assignment(inst.cost, eps)
                    np.testing.assert_array_equal(m.match_of_a, want_t.match_of_a)
                    np.testing.assert_array_equal(s.free_counts, want_t.free_counts)
    finally:
        sv.close()


# ---- degenerate inputs (ties, exact multiples of eps, extreme shapes) ------
@pytest.mark.parametrize("case", ["zeros", "ones", "multiples", "two_values", "single_row",
                                  "single_col"])
def test_degenerate_costs_match_oracle(oracle, case):
    rng = np.random.default_rng(17)
    eps = 0.05
    if case == "zeros":
        cost = np.zeros((300, 300))          # every edge admissible: maximal contention
    elif case == "ones":
        cost = np.ones((257, 200))
    elif case == "multiples":                 # exact multiples of eps (scaled_floor boundaries)
        cost = rng.integers(0, 21, (256, 256)) * eps
        cost = np.minimum(cost, 1.0)
    elif case == "two_values":
        cost = np.where(rng.random((400, 333)) < 0.5, 0.25, 0.75)
    elif case == "single_row":
        cost = rng.random((1, 500))
    else:
        cost = rng.random((500, 1))
    want = oracle.solve_assignment(cost, eps)
    m, s = _solve(otprg.AssignmentInstance(*cost.shape, cost), eps)
    np.testing.assert_array_equal(m.match_of_a, want.match_of_a)
    np.testing.assert_array_equal(s.duals_final.y_a, want.y_a)
    np.testing.assert_array_equal(s.duals_final.y_b, want.y_b)
    np.testing.assert_array_equal(s.free_counts, want.free_counts)
    assert s.device["cost"] == want.cost


# ---- uint32 storage: eps below ~1/65531 ------------------
# The reference accepts any eps with unit_floor + 4 <= INT32_MAX
# (core.cpp:36-41); below uint16's range the device stores kT / t as uint32.

def _assert_same_as_oracle(m, s, want):
    np.testing.assert_array_equal(m.match_of_a, want.match_of_a)
    np.testing.assert_array_equal(m.match_of_b, want.match_of_b)
    np.testing.assert_array_equal(s.duals_final.y_a, want.y_a)
    np.testing.assert_array_equal(s.duals_final.y_b, want.y_b)
    assert s.phases == want.phases and s.sum_ni == want.sum_ni
    np.testing.assert_array_equal(s.free_counts, want.free_counts)
    assert s.device["cost"] == want.cost and s.swapped == want.swapped


def test_one_by_one_tiny_eps_u32():
    eps = 1e-5  # unit_floor 100000: beyond uint16
    m, s = _solve(_single(0.375), eps)
    assert s.device["width"] == 4
    k = otprg.scale_round_costs(_single(0.375), eps).k[0, 0]
    assert s.phases == k + 1 and m.match_of_a[0] == 0
    assert s.duals_final.y_b[0] == k + 1 and s.duals_final.y_a[0] == -1


@pytest.mark.parametrize("n_a,n_b,eps,seed", [(48, 40, 1.0 / 70000.0, 1), (30, 45, 1e-5, 2),
                                              (64, 64, 2e-6, 3)])
def test_tiny_eps_u32_vs_oracle(oracle, n_a, n_b, eps, seed):
    cost = np.random.default_rng(seed).random((n_a, n_b))
    want = oracle.solve_assignment(cost, eps)
    m, s = _solve(otprg.AssignmentInstance(n_a, n_b, cost), eps)
    assert s.device["width"] == 4
    _assert_same_as_oracle(m, s, want)


def test_explicit_storage_too_narrow_is_parameter_error():
    with pytest.raises(otprg.ParameterError):
        _solve(_single(0.5), 1e-5, "u16")
    with pytest.raises(otprg.ParameterError):
        _solve(_single(0.5), 0.001, "u8")


# ---- costs="on_the_fly" through the public API (north star: costs from the
# point coordinates when the matrix would not fit in HBM) ---------------------

def test_public_api_on_the_fly_costs(golden):
    for key in ("square_n10000_eps0.01_s1", "square_n1000_eps0.1_s2", "square_n3000_eps0.02_s1"):
        w = golden[key]
        inst = otprg.gen_uniform_square(w["n_a"], w["seed"])
        m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"], costs="on_the_fly"))
        _assert_matches_golden(key, w, m, s)
        assert s.device.get("n_shards") == 1
    with pytest.raises(otprg.ParameterError):
        otprg.solve_assignment(_single(0.5), otprg.AssignmentOptions(eps=0.1, costs="bogus"))
