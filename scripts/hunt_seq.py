"""Solve golden cases sequentially in ONE process/context (as pytest does),
printing each key before the solve, to find state carried across solves."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import PIN_KEYS, pins_of, random_instance  # noqa: E402

golden = json.load(open("tests/golden/assign_pins.json"))
order = sys.argv[1] if len(sys.argv) > 1 else "random,square"
keys = []
for kind in order.split(","):
    keys += sorted(k for k, v in golden.items() if v["kind"] == kind and v["n_a"] <= 4000)
for key in keys:
    w = golden[key]
    if w["kind"] == "square":
        inst = otprg.gen_uniform_square(w["n_a"], w["seed"])
    else:
        inst = otprg.AssignmentInstance(w["n_a"], w["n_b"], random_instance(w["n_a"], w["n_b"], w["seed"]))
    print("solving", key, flush=True)
    m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"]))
    got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases,
                  s.sum_ni, s.device["cost"])
    print("  ", "OK" if all(got[k] == w[k] for k in PIN_KEYS) else "WRONG", s.phases, flush=True)
