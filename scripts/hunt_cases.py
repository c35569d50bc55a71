"""Run every golden square case (n <= max_n) in its own subprocess with a
timeout; report hangs / wrong results.  Usage: hunt_cases.py [max_n] [lib]"""
import json
import os
import subprocess
import sys

max_n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
golden = json.load(open("tests/golden/assign_pins.json"))
keys = sorted(k for k, v in golden.items() if v["kind"] == "square" and v["n_a"] <= max_n)
code = r'''
import sys, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2203_03732_b200 as otprg
from golden_util import pins_of, PIN_KEYS
key = sys.argv[1]; storage = sys.argv[2]
w = json.load(open("tests/golden/assign_pins.json"))[key]
m, s = otprg.solve_assignment(otprg.gen_uniform_square(w["n_a"], w["seed"]),
                              otprg.AssignmentOptions(eps=w["eps"], storage=storage))
got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni, s.device["cost"])
print("OK" if all(got[k] == w[k] for k in PIN_KEYS) else f"WRONG phases {s.phases} want {w['phases']}")
'''
for key in keys:
    for storage in ("u16", "u8"):
        try:
            r = subprocess.run([sys.executable, "-c", code, key, storage], capture_output=True,
                               text=True, timeout=30, env=os.environ)
            out = (r.stdout.strip().splitlines() or ["?"])[-1] if r.returncode == 0 else \
                "ERR " + r.stderr.strip().splitlines()[-1]
        except subprocess.TimeoutExpired:
            out = "HANG"
        print(key, storage, out, flush=True)
