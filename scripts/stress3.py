"""Repeat a solve and report device errors/bad results (race hunting)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import json  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import pins_of  # noqa: E402

golden = json.load(open("tests/golden/assign_pins.json"))
n, eps, seed, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
key = f"square_n{n}_eps{eps!r}_s{seed}"
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(n, seed), eps)
bad, errs = 0, {}
for r in range(reps):
    try:
        m, s = S.solve_prepared()
        p = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni, s.device["cost"])
        bad += not all(p[k] == golden[key][k] for k in p)
    except Exception as e:
        errs[str(e)[:90]] = errs.get(str(e)[:90], 0) + 1
print(key, "reps", reps, "bad", bad, "errors", errs, flush=True)
