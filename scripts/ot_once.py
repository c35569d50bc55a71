"""One config-5 solve_ot (gen_random_ot_rational(n, n, 1), eps 0.01) — a short command for ncu."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
plan, st = otprg.solve_ot(otprg.gen_random_ot_rational(n, n, 1), 0.01)
print("phases", st.phases, "loop_ms", st.device["loop_ms"], "entries", len(plan.a))
