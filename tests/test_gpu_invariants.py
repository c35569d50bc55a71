"""GPU tests of the device invariant suite and the host-synced observer loop
(reference A12: verify_feasibility assignment.cpp:264-312,
check_invariants :344-349, observer :350-355).

Structure follows the reference's tests/test_assignment.cpp ("verify_feasibility
flags corrupted duals", "per-phase invariants hold on random instances") and
acceptance.cpp's verified_options observer.  The device report is checked
against a plain-Python restatement of verify_feasibility (below: the test's
oracle, in the reference's order of checks)."""
import numpy as np
import pytest

from golden_util import PIN_KEYS, pins_of, random_instance

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")


def py_verify(k, ya, yb, ma, mb, unit_ceil):
    """assignment.cpp:264-312 + core.cpp:69-86, every violation in order."""
    n_a, n_b = k.shape
    for a in range(n_a):
        b = ma[a]
        if b != -1 and (b < 0 or b >= n_b or mb[b] != a):
            return [f"matching is not mutually consistent at a={a}"]
    for b in range(n_b):
        a = mb[b]
        if a != -1 and (a < 0 or a >= n_a or ma[a] != b):
            return [f"matching is not mutually consistent at b={b}"]
    bound = unit_ceil + 2
    out = []
    for a in range(n_a):
        if ya[a] > 0:
            out.append(f"demand dual positive at a={a}")
        if ma[a] == -1 and ya[a] != 0:
            out.append(f"free demand vertex with nonzero dual at a={a}")
        if abs(ya[a]) > bound:
            out.append(f"demand dual magnitude exceeds bound at a={a}")
    for b in range(n_b):
        if yb[b] < 0:
            out.append(f"supply dual negative at b={b}")
        if abs(yb[b]) > bound:
            out.append(f"supply dual magnitude exceeds bound at b={b}")
    s = ya[:, None] + yb[None, :]
    for a, b in zip(*np.nonzero((s != k) | (s > k + 1))):
        if ma[a] == b:
            if s[a, b] != k[a, b]:
                out.append(f"matching edge not tight at ({a},{b}): Y(a)+Y(b)={s[a, b]} k={k[a, b]}")
        elif s[a, b] > k[a, b] + 1:
            out.append(f"dual sum exceeds rounded cost allowance at ({a},{b}): "
                       f"Y(a)+Y(b)={s[a, b]} k={k[a, b]}")
    return out


def _same(rep, want):
    assert rep.ok() == (not want)
    if want:
        assert rep.violations[0] == want[0]
        assert rep.count == len(want)


def test_verify_flags_corrupted_duals():
    """test_assignment.cpp:258-265."""
    inst = otprg.AssignmentInstance(4, 4, random_instance(4, 4, 9))
    sc = otprg.scale_round_costs(inst, 0.2)
    m = otprg.Matching.empty(4, 4)
    d = otprg.DualState(np.zeros(4, np.int64), np.ones(4, np.int64))
    assert otprg.verify_feasibility(sc, d, m).ok()
    d.y_b[2] += 10
    rep = otprg.verify_feasibility(sc, d, m)
    assert not rep.ok()
    _same(rep, py_verify(sc.k, d.y_a, d.y_b, m.match_of_a, m.match_of_b, sc.unit_ceil))


def test_verify_random_corruptions_match_restatement():
    rng = np.random.default_rng(3)
    inst = otprg.AssignmentInstance(50, 40, random_instance(50, 40, 5))
    eps = 0.05
    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps))
    sc = otprg.scale_round_costs(inst, eps)
    # base: the completed matching with the final duals (itself usually not
    # feasible: completion pairs are not tight), then random corruptions
    base_ma, base_mb = m.match_of_a.copy(), m.match_of_b.copy()
    ya, yb = s.duals_final.y_a.astype(np.int64), s.duals_final.y_b.astype(np.int64)
    for trial in range(40):
        ma, mb, a_, b_ = base_ma.copy(), base_mb.copy(), ya.copy(), yb.copy()
        kind = trial % 5
        if kind == 0:
            a_[rng.integers(50)] += int(rng.integers(1, 4))
        elif kind == 1:
            b_[rng.integers(40)] -= int(rng.integers(1, 30))
        elif kind == 2:
            b_[rng.integers(40)] += int(rng.integers(1, 30))
        elif kind == 3:
            a = int(rng.integers(50))
            ma[a] = (ma[a] + 1) % 40
        else:
            a_[rng.integers(50)] -= int(rng.integers(1, 50))
        rep = otprg.verify_feasibility(sc, otprg.DualState(a_, b_), otprg.Matching(ma, mb))
        _same(rep, py_verify(sc.k, a_, b_, ma, mb, sc.unit_ceil))


def _maximality(snap):
    """acceptance.cpp:113-123 / test_assignment.cpp check_maximality."""
    prime_a = {a for a, _ in snap.workset.m_prime}
    prime_b = {b for _, b in snap.workset.m_prime}
    for i, b in enumerate(snap.workset.b_free):
        if b in prime_b:
            continue
        for a in snap.workset.e_admissible[i]:
            assert a in prime_a, f"phase {snap.phase}: b={b} left free with free admissible a={a}"


def _greedy_from_workset(ws):
    """The reference's sequential greedy (assignment.cpp:161-171) replayed on
    the exported E': must reproduce the device's M' exactly."""
    claimed, out = set(), []
    for i, b in enumerate(ws.b_free):
        for a in ws.e_admissible[i]:
            if a not in claimed:
                claimed.add(int(a))
                out.append((int(a), int(b)))
                break
    return out


def _observer(n_a, n_b, eps, log):
    state = {"matched": 0}

    def obs(snap):
        bound = snap.costs.unit_ceil + 2
        ya, yb = snap.duals.y_a, snap.duals.y_b
        assert (ya <= 0).all() and (yb >= 0).all()
        free_a = snap.matching.match_of_a == -1
        assert (ya[free_a] == 0).all()
        assert (np.abs(ya) <= bound).all() and (np.abs(yb) <= bound).all()
        matched = snap.matching.size()
        assert matched >= state["matched"]
        state["matched"] = matched
        assert snap.sum_abs_after - snap.sum_abs_before >= len(snap.workset.b_free)
        _maximality(snap)
        assert snap.workset.m_prime == _greedy_from_workset(snap.workset)
        log.append(snap.phase)

    return obs


def test_per_phase_invariants_random_instances(golden):
    """test_assignment.cpp:267-303 (seeds 1..8, 30x30, eps 0.08/0.15) with the
    device suite after every phase; results bit-exact with the golden pins."""
    for seed in range(1, 9):
        eps = 0.15 if seed % 2 == 0 else 0.08
        inst = otprg.AssignmentInstance(30, 30, random_instance(30, 30, seed * 131))
        log = []
        opt = otprg.AssignmentOptions(eps=eps, check_invariants=True, observer=_observer(30, 30, eps, log))
        m, s = otprg.solve_assignment(inst, opt)
        assert m.size() == 30
        assert s.phases <= s.phase_bound(eps)
        assert s.sum_ni <= s.sum_ni_bound(eps, 30)
        assert log == list(range(1, s.phases + 1))
        key = f"random_30x30_eps{eps!r}_s{seed * 131}"
        if key in golden:
            got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts,
                          s.phases, s.sum_ni, s.device["cost"])
            assert {k: got[k] for k in PIN_KEYS} == {k: golden[key][k] for k in PIN_KEYS}


def test_observer_admissible_sets_match_restatement():
    """E' exported from the device equals the admissible sets recomputed from
    the snapshot's costs and the previous phase's duals."""
    inst = otprg.gen_uniform_square(300, 2, dense=True)
    eps = 0.02
    prev = {}

    def obs(snap):
        k = snap.costs.k
        if prev:
            ya, yb = prev["ya"], prev["yb"]
            for i, b in enumerate(snap.workset.b_free):
                want = np.flatnonzero(ya + yb[b] == k[:, b] + 1)
                assert np.array_equal(snap.workset.e_admissible[i], want), (snap.phase, b)
        prev["ya"], prev["yb"] = snap.duals.y_a.copy(), snap.duals.y_b.copy()

    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps, observer=obs))
    m2, s2 = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps))
    assert np.array_equal(m.match_of_a, m2.match_of_a) and s.phases == s2.phases


@pytest.mark.parametrize("key", ["square_n2000_eps0.01_s3", "square_n10000_eps0.01_s1"])
def test_check_invariants_at_scale(golden, key):
    """Acceptance criteria 4/5 as a GPU gate: the full feasibility check after
    every phase at n = 2,000 (1,547 phases) and n = 10,000 (config 2)."""
    w = golden[key]
    inst = otprg.gen_uniform_square(w["n_a"], w["seed"])
    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"], check_invariants=True))
    got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                  s.sum_ni, s.device["cost"])
    assert {k: got[k] for k in PIN_KEYS} == {k: w[k] for k in PIN_KEYS}


def test_swapped_orientation_observer():
    inst = otprg.AssignmentInstance(5, 12, random_instance(5, 12, 78))
    seen = []

    def obs(snap):
        assert snap.costs.k.shape == (12, 5)  # internal orientation: n_a >= n_b
        assert len(snap.matching.match_of_a) == 12
        seen.append(snap.phase)

    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.1, check_invariants=True,
                                                                observer=obs))
    assert s.swapped and m.size() == 5 and seen == list(range(1, s.phases + 1))


@pytest.mark.parametrize("storage", ["u8", "u16", "u32"])
@pytest.mark.parametrize("shape", [(60, 60), (70, 45), (45, 70)])
def test_state_verify_matches_restatement_after_completion(storage, shape):
    """The solver-state kernels (packed SIMD over the B-major kT) against the
    restatement on a state that HAS violations: the completed matching (the
    index-order completion pairs are generally not tight) with the final
    duals, and on the clean state of every phase."""
    n_a, n_b = shape
    inst = otprg.AssignmentInstance(n_a, n_b, random_instance(n_a, n_b, 11))
    eps = 0.1
    swapped = n_b > n_a
    sv = otprg.Solver(0)
    sc = sv.scale_round_costs(inst, eps, storage)
    k = np.ascontiguousarray(sc.k.T) if swapped else sc.k
    sv._prepared = (n_a, n_b, eps)
    sv.begin()
    phase = 0
    while True:
        done, fin = sv.step(phase + 1)
        if done == phase:
            break
        phase = done
        m, s = sv.snapshot()
        mi = otprg.Matching(m.match_of_b, m.match_of_a) if swapped else m
        want = py_verify(k, s.duals_final.y_a, s.duals_final.y_b, mi.match_of_a, mi.match_of_b,
                         sc.unit_ceil)
        _same(sv.verify_feasibility(), want)
        assert not want
    m, s = sv.finish()
    mi = otprg.Matching(m.match_of_b, m.match_of_a) if swapped else m
    want = py_verify(k, s.duals_final.y_a, s.duals_final.y_b, mi.match_of_a, mi.match_of_b,
                     sc.unit_ceil)
    _same(sv.verify_feasibility(), want)
    sv.close()
