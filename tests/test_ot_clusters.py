"""CPU tests of the copy/cluster host checks (check_cluster_invariant /
check_cluster_feasibility, ot.cpp:190-315) and plan_from_flow (ot.cpp:639-703)
of libotprg.so: the reference's final states (tests/golden/copy_*.npz) pass,
and on corrupted states the violation lists equal the UNMODIFIED reference's,
message for message."""
import os

import numpy as np
import pytest

import paper_2203_03732_b200 as otprg
from oracle.pyoracle import FLAT_KEYS

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_group(group):
    with np.load(os.path.join(GOLDEN, f"copy_{group}.npz")) as z:
        cases = {}
        for key in z.files:
            i, name = key.split("_", 1)
            cases.setdefault(int(i), {})[name] = z[key]
    return [cases[i] for i in sorted(cases)]


def copy_instance(c):
    return otprg.CopyInstance(otprg.ScaledCosts(float(c["eps"]), c["k"], int(c["unit_floor"]),
                                                int(c["unit_ceil"])), c["demand_copies"], c["supply_copies"])


def state_of(flat):
    """Flat arrays (include/otprg.h layout) -> ClusterState."""
    dem_off, flow_off, sup_off = flat["dem_off"], flat["flow_off"], flat["sup_off"]
    demand = [[otprg.DemandCluster(int(flat["dem_y"][c]), int(flat["dem_free"][c]),
                                   [(int(flat["flow_b"][f]), int(flat["flow_cnt"][f]))
                                    for f in range(int(flow_off[c]), int(flow_off[c + 1]))])
               for c in range(int(dem_off[a]), int(dem_off[a + 1]))] for a in range(len(dem_off) - 1)]
    supply = [[otprg.SupplyCluster(int(flat["sup_y"][c]), int(flat["sup_free"][c]), int(flat["sup_matched"][c]))
               for c in range(int(sup_off[b]), int(sup_off[b + 1]))] for b in range(len(sup_off) - 1)]
    return otprg.ClusterState(demand, supply)


def flat_of(state):
    st, keep = state._c()
    return dict(zip(FLAT_KEYS, keep))


@pytest.mark.parametrize("group", ["micro", "larger", "wide"])
def test_reference_final_states_pass_checks(group):
    for c in load_group(group):
        st = state_of({x: c[f"state_{x}"] for x in FLAT_KEYS})
        inst = copy_instance(c)
        assert otprg.check_cluster_invariant(st, inst).ok()
        assert otprg.check_cluster_feasibility(st, inst).ok()


def _corruptions(st, rng):
    """A few single-point corruptions of a valid state (new ClusterState each)."""
    import copy
    out = []
    live_d = [(a, i) for a, cs in enumerate(st.demand) for i in range(len(cs))]
    live_s = [(b, i) for b, cs in enumerate(st.supply) for i in range(len(cs))]
    for _ in range(6):
        s2 = copy.deepcopy(st)
        kind = int(rng.integers(0, 8))
        if kind == 0 and live_d:  # shift a demand dual
            a, i = live_d[int(rng.integers(len(live_d)))]
            s2.demand[a][i].y += int(rng.choice([-2, -1, 1]))
        elif kind == 1 and live_s:  # shift a supply dual
            b, i = live_s[int(rng.integers(len(live_s)))]
            s2.supply[b][i].y += int(rng.choice([-3, -1, 1, 2]))
        elif kind == 2 and live_d:  # extra free demand copy
            a, i = live_d[int(rng.integers(len(live_d)))]
            s2.demand[a][i].free_count += 1
        elif kind == 3 and live_s:  # matched -> free on the supply side
            b, i = live_s[int(rng.integers(len(live_s)))]
            if s2.supply[b][i].matched_count:
                s2.supply[b][i].matched_count -= 1
                s2.supply[b][i].free_count += 1
        elif kind == 4 and live_d:  # third dual on a demand vertex
            a, _ = live_d[int(rng.integers(len(live_d)))]
            s2.demand[a].append(otprg.DemandCluster(-7, 1, []))
        elif kind == 5 and live_s:  # free supply split across duals
            b, _ = live_s[int(rng.integers(len(live_s)))]
            s2.supply[b].append(otprg.SupplyCluster(-1, 2, 0))
        elif kind == 6 and live_d:  # flow moved to another b
            a, i = live_d[int(rng.integers(len(live_d)))]
            if s2.demand[a][i].flow:
                b, cnt = s2.demand[a][i].flow[0]
                s2.demand[a][i].flow[0] = ((b + 1) % len(st.supply), cnt)
        elif kind == 7 and live_d:  # huge dual
            a, i = live_d[int(rng.integers(len(live_d)))]
            s2.demand[a][i].y = -10_000
        out.append(s2)
    return out


@pytest.mark.parametrize("group", ["micro", "larger", "wide"])
def test_check_messages_match_reference_on_corrupted_states(reference, group):
    rng = np.random.default_rng(5)
    n = 0
    for c in load_group(group):
        base = state_of({x: c[f"state_{x}"] for x in FLAT_KEYS})
        inst = copy_instance(c)
        for st in _corruptions(base, rng):
            for which, fn in ((0, otprg.check_cluster_invariant), (1, otprg.check_cluster_feasibility)):
                got = fn(st, inst).violations
                want = reference.check_cluster(c["k"], int(c["unit_ceil"]), c["demand_copies"],
                                               c["supply_copies"], flat_of(st), which)
                assert got == want, (group, which)
                n += bool(want)
    assert n > 0  # the corruptions really were caught


def test_plan_from_flow_matches_solve_ot_reference_plans(reference):
    """plan_from_flow on the reference's own copy flow reproduces the
    reference's solve_ot plan bit for bit (ot.cpp:705-732 composition)."""
    for n_a, n_b, seed, eps in ((6, 4, 3, 0.23), (10, 10, 7, 0.25), (30, 20, 5, 0.1)):
        inst = otprg.gen_random_ot_rational(n_a, n_b, seed)
        sm = otprg.scale_and_round(inst, eps / 3.0)
        k, uf, uc = reference.scale_round_costs(inst.cost, eps / 3.0)
        r = reference.solve_copy_matching(k, eps / 3.0, uf, uc, sm.d, sm.s, eps / 3.0, check=False,
                                          phase_cap=1)
        plan = otprg.plan_from_flow(r["flow"], sm, inst)
        want = reference.solve_ot(inst.mu, inst.nu, inst.cost, eps)
        assert plan.cost == want["cost"]
        np.testing.assert_array_equal(plan.a, want["a"])
        np.testing.assert_array_equal(plan.b, want["b"])
        assert plan.mass.tobytes() == want["mass"].tobytes()
