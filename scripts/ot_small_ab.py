"""OT loop time of the host-sized phases (OTPRG_OT_HOST_SIZED=1), the device-sized
phase as a launch sequence (OTPRG_OT_SEQ=1) and the persistent phase loop (default),
small and config-5 instances, plan bits compared."""
import os
import subprocess
import sys

code = r'''
import sys, hashlib
sys.path.insert(0, ".")
import numpy as np
import paper_2203_03732_b200 as otprg
n, eps = int(sys.argv[1]), float(sys.argv[2])
inst = otprg.gen_random_ot_rational(n, n, 1)
best = None
for rep in range(4):
    plan, st = otprg.solve_ot(inst, eps)
    best = st.device["loop_ms"] if best is None else min(best, st.device["loop_ms"])
h = hashlib.sha1(np.asarray(plan.a).tobytes() + np.asarray(plan.b).tobytes() + np.asarray(plan.mass).tobytes()
                 + float(plan.cost).hex().encode()).hexdigest()[:12]
print(f"n={n} eps={eps} phases={st.phases} loop_ms={best:.2f} plan={h}")
'''
for n, eps in ((100, 0.01), (1000, 0.01), (5000, 0.01), (20000, 0.01)):
    for mode in ("host", "seq", "persistent"):
        env = dict(os.environ, OTPRG_OT_PROFILE="1")
        if mode == "host":
            env["OTPRG_OT_HOST_SIZED"] = "1"
        if mode == "seq":
            env["OTPRG_OT_SEQ"] = "1"
        r = subprocess.run([sys.executable, "-c", code, str(n), str(eps)], env=env, capture_output=True, text=True)
        err = [l for l in r.stderr.splitlines() if "ot loop" in l or "Error" in l]
        print(mode, r.stdout.strip(), err[-1] if err else r.stderr[-300:], flush=True)
