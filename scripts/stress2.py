"""Compare solve_prepared vs the stepping API (race hunting)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import json  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import pins_of  # noqa: E402

golden = json.load(open("tests/golden/assign_pins.json"))
n, eps, seed = 4000, 0.01, 1
key = f"square_n{n}_eps{eps!r}_s{seed}"
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(n, seed), eps)


def ok(m, s):
    p = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni, s.device["cost"])
    return all(p[k] == golden[key][k] for k in p), tuple(s.free_counts[:3])


for mode in ("solve", "step1_then_all", "all_at_once", "solve"):
    bad = []
    for r in range(15):
        if mode == "solve":
            m, s = S.solve_prepared()
        else:
            S.begin()
            if mode == "step1_then_all":
                S.step(1)
            m, s = S.finish()
        good, fc = ok(m, s)
        if not good:
            bad.append(fc)
    print(mode, "bad", len(bad), bad[:3], flush=True)
