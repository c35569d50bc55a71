"""Repeat solves and report result variability (race detector)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import json  # noqa: E402
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import pins_of  # noqa: E402

golden = json.load(open("tests/golden/assign_pins.json"))
cases = [(4000, 0.01, 1), (3000, 0.02, 1), (2000, 0.01, 3), (1000, 0.01, 2)]
S = otprg.Solver(0)
for n, eps, seed in cases:
    key = f"square_n{n}_eps{eps!r}_s{seed}"
    inst = otprg.gen_uniform_square(n, seed)
    S.prepare(inst, eps)
    bad = 0
    fcs = set()
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
        m, s = S.solve_prepared()
        p = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni, s.device["cost"])
        ok = all(p[k] == golden[key][k] for k in p)
        bad += not ok
        if not ok:
            fcs.add(tuple(s.free_counts[:4]))
    print(key, "bad", bad, "examples", list(fcs)[:3], flush=True)
