"""The copy/cluster solver on the device (solve_copy_matching, ot.cpp:418-637;
OTOptions hooks, ot.hpp:124-156) against the UNMODIFIED reference's fixtures
(tests/golden/copy_*.npz, make_golden_copy.py): phase counts, free_counts,
the flow after EVERY phase (observer), the final flow and the final
ClusterState, with check_invariants on.  Then, as tests/test_ot.cpp:234-346,
the compressed solver against the explicit copy solver (device copy mode)
phase by phase.  Bit-exact throughout."""
import numpy as np
import pytest

from test_ot_clusters import copy_instance, flat_of, load_group

pytestmark = pytest.mark.gpu
otprg = pytest.importorskip("paper_2203_03732_b200")


def _solve_recording(c, check=True):
    flows, nis, sums = [], [], []

    def obs(snap):
        flows.append(snap.state.flow_matrix(*c["k"].shape))
        nis.append(snap.n_i)
        sums.append((snap.sum_abs_before, snap.sum_abs_after, snap.state.sum_abs_duals()))
        assert snap.phase == len(flows)
        np.testing.assert_array_equal(snap.inst.costs.k, c["k"])

    res = otprg.solve_copy_matching(copy_instance(c), float(c["eps"]),
                                    otprg.ClusterOptions(check_invariants=check, observer=obs))
    return res, flows, nis, sums


@pytest.mark.parametrize("group", ["micro", "larger", "wide"])
def test_copy_matching_matches_reference_every_phase(group):
    for i, c in enumerate(load_group(group)):
        res, flows, nis, sums = _solve_recording(c)
        assert res.stats.phases == int(c["phases"]), (group, i)
        np.testing.assert_array_equal(res.stats.free_counts, c["free_counts"])
        assert res.stats.sum_ni == int(c["sum_ni"])
        assert bool(res.stats.full_match_termination) == bool(c["full_match_termination"])
        np.testing.assert_array_equal(res.flow, c["flow"])
        got = flat_of(res.state)
        for x, v in got.items():
            np.testing.assert_array_equal(v, c[f"state_{x}"], err_msg=f"{group} {i} {x}")
        npf = len(c["phase_flows"])
        assert len(flows) == int(c["phases"])
        np.testing.assert_array_equal(np.array(flows[:npf]), c["phase_flows"])
        np.testing.assert_array_equal(np.array(nis[:npf]), c["phase_ni"])
        for before, after, now in sums:
            assert after == now and before >= 0


def _explicit_phase_flows(c):
    """The explicit copy solver (copy mode, assignment.cpp:81-103/241-250) on
    materialised copies of the same rounded costs, flows per phase."""
    k, eps = c["k"], float(c["eps"])
    cost = k.astype(np.float64) * eps  # RN(k eps): scale_round_costs gives back k
    dg = np.repeat(np.arange(len(c["demand_copies"])), c["demand_copies"]).astype(np.int32)
    sg = np.repeat(np.arange(len(c["supply_copies"])), c["supply_copies"]).astype(np.int32)
    cc = cost[np.ix_(dg, sg)]
    n_a, n_b = k.shape
    flows, nis = [], []

    def fl(ma):
        f = np.zeros((n_a, n_b), np.int64)
        for a2, b2 in enumerate(ma):
            if b2 >= 0:
                f[dg[a2], sg[b2]] += 1
        return f

    def obs(snap):
        flows.append(fl(snap.matching.match_of_a))
        nis.append(len(snap.workset.b_free))

    inst = otprg.AssignmentInstance(*cc.shape, cc)
    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps, demand_groups=dg, supply_groups=sg,
                                                                check_invariants=True, observer=obs))
    assert not s.swapped
    return flows, nis, fl(m.match_of_a), s


@pytest.mark.parametrize("group", ["micro", "larger"])
def test_compressed_equals_explicit_phase_by_phase(group):
    for c in load_group(group):
        assert np.array_equal(otprg.scale_round_costs(
            otprg.AssignmentInstance(*c["k"].shape, c["k"].astype(np.float64) * float(c["eps"])),
            float(c["eps"])).k, c["k"])
        res, flows, nis, _ = _solve_recording(c)
        eflows, enis, efinal, es = _explicit_phase_flows(c)
        assert res.stats.phases == es.phases
        assert nis == enis
        for p in range(len(flows)):
            np.testing.assert_array_equal(flows[p], eflows[p])
        np.testing.assert_array_equal(res.flow, efinal)


def test_observer_exception_propagates():
    c = load_group("larger")[0]

    class Stop(Exception):
        pass

    def obs(snap):
        if snap.phase == 1:
            raise Stop()

    with pytest.raises(Stop):
        otprg.solve_copy_matching(copy_instance(c), float(c["eps"]), otprg.ClusterOptions(observer=obs))


def test_copy_instance_validation():
    c = load_group("micro")[0]
    inst = copy_instance(c)
    bad = otprg.CopyInstance(inst.costs, inst.demand_copies, inst.supply_copies + 100)
    with pytest.raises(otprg.ParameterError):
        otprg.solve_copy_matching(bad, 0.2)
    neg = otprg.CopyInstance(inst.costs, -inst.demand_copies, inst.supply_copies)
    with pytest.raises(otprg.ParameterError):
        otprg.solve_copy_matching(neg, 0.2)
    with pytest.raises(otprg.ParameterError):
        otprg.solve_copy_matching(inst, 1.0)


def test_solve_ot_hooks_do_not_change_the_result():
    """OTOptions (ot.hpp:153-156): check_invariants + observer on solve_ot give
    the same plan / stats; the observer sees every phase with n_i =
    free_counts and the CopyInstance at eps/3; the last state passes the checks."""
    for n_a, n_b, seed, eps in ((6, 4, 3, 0.23), (10, 10, 7, 0.25), (50, 50, 1, 0.1)):
        inst = otprg.gen_random_ot_rational(n_a, n_b, seed)
        plan0, st0 = otprg.solve_ot(inst, eps)
        seen = []
        plan, st = otprg.solve_ot(inst, eps, otprg.OTOptions(check_invariants=True,
                                                             observer=lambda s: seen.append(s)))
        assert plan.cost == plan0.cost and plan.mass.tobytes() == plan0.mass.tobytes()
        np.testing.assert_array_equal(plan.a, plan0.a)
        np.testing.assert_array_equal(st.free_counts, st0.free_counts)
        assert [s.phase for s in seen] == list(range(1, st.phases + 1))
        assert [s.n_i for s in seen] == list(st.free_counts)
        sm = otprg.scale_and_round(inst, eps / 3.0)
        np.testing.assert_array_equal(seen[0].inst.demand_copies, sm.d)
        np.testing.assert_array_equal(seen[0].inst.costs.k,
                                      otprg.scale_round_costs(otprg.AssignmentInstance(n_a, n_b, inst.cost),
                                                              eps / 3.0).k)
        last = otprg.last_cluster_state()
        assert otprg.check_cluster_invariant(last, seen[-1].inst).ok()
        assert otprg.check_cluster_feasibility(last, seen[-1].inst).ok()


def test_plan_from_flow_reproduces_solve_ot():
    """solve_ot = scale_and_round -> solve_copy_matching(eps/3) -> plan_from_flow."""
    for n_a, n_b, seed, eps in ((10, 10, 14, 0.1), (100, 100, 1, 0.1)):
        inst = otprg.gen_random_ot_rational(n_a, n_b, seed)
        plan0, st0 = otprg.solve_ot(inst, eps)
        sm = otprg.scale_and_round(inst, eps / 3.0)
        sc = otprg.scale_round_costs(otprg.AssignmentInstance(n_a, n_b, inst.cost), eps / 3.0)
        ci = otprg.CopyInstance(sc, sm.d, sm.s)
        res = otprg.solve_copy_matching(ci, eps / 3.0)
        np.testing.assert_array_equal(res.stats.free_counts, st0.free_counts)
        plan = otprg.plan_from_flow(res.flow, sm, inst)
        assert plan.cost == plan0.cost and plan.mass.tobytes() == plan0.mass.tobytes()
