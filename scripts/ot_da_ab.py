"""A/B of the OT DA round paths: OTPRG_OT_DA_BATCH = 0 (sorted, one sync per
round) against device-sized batches; loop time of config 5 and a small case,
plan bits compared."""
import os
import subprocess
import sys

code = r'''
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2203_03732_b200 as otprg
n = int(sys.argv[1])
inst = otprg.gen_random_ot_rational(n, n, 1)
best = None
for rep in range(4):
    plan, st = otprg.solve_ot(inst, 0.01)
    best = st.device["loop_ms"] if best is None else min(best, st.device["loop_ms"])
h = hash((tuple(np.asarray(plan.a).tolist()), tuple(np.asarray(plan.b).tolist()), tuple(np.asarray(plan.mass).tolist()), plan.cost))
print(f"n={n} phases={st.phases} loop_ms={best:.2f} hash={h}")
'''
for n in (1000, 20000):
    for b in ("0", "1", "2", "4", "8"):
        env = dict(os.environ, OTPRG_OT_DA_BATCH=b, OTPRG_OT_PROFILE="1")
        r = subprocess.run([sys.executable, "-c", code, str(n)], env=env, capture_output=True, text=True)
        err = [l for l in r.stderr.splitlines() if "ot loop" in l or "Error" in l]
        print("batch", b, r.stdout.strip(), err[-1] if err else "", flush=True)
