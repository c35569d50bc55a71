"""Runs the Python examples of INTEGRATION.md (smaller sizes) and checks the claims they make."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

inst = otprg.gen_uniform_square(3000, seed=1)
m, stats = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.01))
m2, stats2 = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.01, costs="on_the_fly"))
assert (m.match_of_a == m2.match_of_a).all() and stats.phases == stats2.phases
opt = otprg.AssignmentOptions(eps=0.01, check_invariants=True, observer=lambda snap: None)
otprg.solve_assignment(inst, opt)
ot = otprg.gen_random_ot_rational(800, 800, seed=1)
plan, st = otprg.solve_ot(ot, eps=0.01)
seen = []
plan_h, _ = otprg.solve_ot(ot, eps=0.01, opt=otprg.OTOptions(check_invariants=True,
                                                              observer=lambda snap: seen.append(snap.n_i)))
assert plan_h.cost == plan.cost and seen == list(st.free_counts)
sm = otprg.scale_and_round(ot, 0.01 / 3)
sc = otprg.scale_round_costs(otprg.AssignmentInstance(800, 800, ot.cost), 0.01 / 3)
ci = otprg.CopyInstance(sc, sm.d, sm.s)
res = otprg.solve_copy_matching(ci, 0.01 / 3)
plan2 = otprg.plan_from_flow(res.flow, sm, ot)
assert plan2.cost == plan.cost and plan2.mass.tobytes() == plan.mass.tobytes()
assert otprg.check_cluster_invariant(res.state, ci).ok()
print("INTEGRATION examples OK")
