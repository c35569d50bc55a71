"""Config 4's code paths pinned to the reference ("pin n <= 20k
runs of the same code path against the oracle").

* n = 20,000, eps = 0.01 (the largest size the reference runs here: 1-2 min
  and 4.8 GB per seed): the fused single-GPU solver, the sharded solver
  (G = 1/2/4/8 logical shards, K = 1/16, u8/u16/u32 slabs) and the on-the-fly
  scans must reproduce tests/golden/assign20k_pins.json (made by the
  UNMODIFIED reference, tests/golden/make_golden_20k.py) bit for bit.
* n = 100,000 (no oracle finishes it): the device verify_feasibility
  (assignment.cpp:264-312) on the pre-completion state of the fused, sharded
  and on-the-fly solves, plus the Lemma bounds phases <= phase_bound(eps)
  and sum_ni <= sum_ni_bound(eps, n) (SolveStats, assignment.cpp:39-52), plus
  bit-identity of the three paths.
"""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN, PIN_KEYS, pins_of

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")
from paper_2203_03732_b200 import sharded  # noqa: E402


@pytest.fixture(scope="module")
def pins20k():
    with open(os.path.join(GOLDEN, "assign20k_pins.json")) as f:
        return json.load(f)


def _check(pins, key, m, s):
    want = pins[key]
    got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                  s.sum_ni, s.device["cost"])
    assert {k: got[k] for k in PIN_KEYS} == {k: want[k] for k in PIN_KEYS}, key
    assert bool(s.full_match_termination) == bool(want["full_match_termination"])


KEYS = ["square_n20000_eps0.01_s1", "square_n20000_eps0.01_s2"]


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("storage", ["u8", "u16", "u32"])
def test_fused_20k(pins20k, key, storage):
    v = pins20k[key]
    m, s = otprg.Solver(0).solve(otprg.gen_uniform_square(v["n_a"], v["seed"]),
                                 otprg.AssignmentOptions(eps=v["eps"], storage=storage))
    _check(pins20k, key, m, s)


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("G,K", [(1, 16), (2, 16), (4, 1), (8, 16), (8, 1), (3, 4)])
@pytest.mark.parametrize("resident", [True, False])
def test_sharded_20k(pins20k, key, G, K, resident):
    v = pins20k[key]
    m, s = sharded.solve_assignment_sharded(otprg.gen_uniform_square(v["n_a"], v["seed"]),
                                            otprg.AssignmentOptions(eps=v["eps"]), G, K=K, resident=resident)
    _check(pins20k, key, m, s)


@pytest.mark.parametrize("storage", ["u8", "u32"])
def test_sharded_20k_storage(pins20k, storage):
    key = KEYS[1]
    v = pins20k[key]
    m, s = sharded.solve_assignment_sharded(otprg.gen_uniform_square(v["n_a"], v["seed"]),
                                            otprg.AssignmentOptions(eps=v["eps"], storage=storage), 4, K=16)
    _check(pins20k, key, m, s)


@pytest.mark.parametrize("key", KEYS)
@pytest.mark.parametrize("G,K,storage", [(1, 16, "u16"), (1, 1, "u16"), (1, 4, "u8"), (2, 4, "u32"),
                                         (2, 1, "u16"), (8, 16, "u16")])
def test_on_the_fly_20k(pins20k, key, G, K, storage):
    """Mid-size on-the-fly parity: at G = 1 the 20k-point shard
    takes the tiled kernel's cross-block split (tsegs > 1) and its merge."""
    v = pins20k[key]
    m, s = sharded.solve_assignment_sharded(otprg.gen_uniform_square(v["n_a"], v["seed"]),
                                            otprg.AssignmentOptions(eps=v["eps"], storage=storage), G,
                                            K=K, on_the_fly=True)
    _check(pins20k, key, m, s)


def _same(a, b):
    (m1, s1), (m2, s2) = a, b
    assert np.array_equal(m1.match_of_a, m2.match_of_a)
    assert np.array_equal(m1.match_of_b, m2.match_of_b)
    assert np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
    assert np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b)
    assert np.array_equal(s1.free_counts, s2.free_counts)
    assert s1.phases == s2.phases and s1.sum_ni == s2.sum_ni


@pytest.mark.slow
def test_100k_feasibility_and_bounds():
    n, eps = 100_000, 0.01
    inst = otprg.gen_uniform_square(n, 1)
    opt = otprg.AssignmentOptions(eps=eps)
    sv = otprg.Solver(0)
    sv.prepare(inst, eps)
    sv.begin()
    sv.step(0)  # every phase, state kept before completion
    rep = sv.verify_feasibility()  # device suite on the solver's own state
    assert rep.ok(), rep.violations
    pre_fused = sv.snapshot()
    fused = sv.finish()
    m, s = fused
    assert s.phases <= otprg.SolveStats.phase_bound(eps)
    assert s.sum_ni <= otprg.SolveStats.sum_ni_bound(eps, n)
    assert m.size() == n and s.phases > 0
    # the sharded and on-the-fly results, checked against the fused context's kT
    for G, otf in ((8, False), (1, True)):
        sv2 = sharded.ShardedSolver(inst, opt, G, K=16, on_the_fly=otf, resident=False)
        try:
            m2, s2, pre = sv2.solve(keep_state=True)
        finally:
            sv2.close()
        rep2 = sv.verify_result(pre[1].duals_final, pre[0])
        assert rep2.ok(), (G, otf, rep2.violations)
        _same(fused, (m2, s2))
        _same(pre_fused, pre)
    # a corrupted state is caught (the check is not vacuous)
    ya = pre_fused[1].duals_final.y_a.copy()
    a = int(np.flatnonzero(pre_fused[0].match_of_a >= 0)[0])
    ya[a] -= 1  # matched edge no longer tight
    bad = sv.verify_result(otprg.DualState(ya, pre_fused[1].duals_final.y_b), pre_fused[0])
    assert not bad.ok()
    sv.close()
