import sys, json, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2203_03732_b200 as otprg
from golden_util import random_instance
g = json.load(open("tests/golden/assign_pins.json"))
for key in sorted(k for k, v in g.items() if v["kind"] == "random"):
    w = g[key]
    inst = otprg.AssignmentInstance(w["n_a"], w["n_b"], random_instance(w["n_a"], w["n_b"], w["seed"]))
    try:
        m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=w["eps"]))
        print(key, "ok", s.phases, flush=True)
    except Exception as e:
        print(key, w["n_a"], w["n_b"], w["eps"], "ERR", e, flush=True)
