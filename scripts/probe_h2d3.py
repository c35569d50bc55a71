"""Pageable 3.2 GB H2D (config 5's cost matrix) through the OT build: build_ms
(H2D + K1 rounding) for OTPRG_H2D_THREADS = 8 .. 48, best of 3; host cores."""
import os
import subprocess
import sys

code = r'''
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg
inst = otprg.gen_random_ot_rational(20000, 20000, 1)
ts = [otprg.solve_ot(inst, 0.01)[1].device["build_ms"] for _ in range(3)]
print(f"{min(ts):.1f}")
'''
print("host cores", os.cpu_count(), flush=True)
for t in (8, 16, 24, 32, 48):
    env = dict(os.environ, OTPRG_H2D_THREADS=str(t))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"threads {t}: build_ms {r.stdout.strip()} {r.stderr[-200:] if r.returncode else ''}", flush=True)
