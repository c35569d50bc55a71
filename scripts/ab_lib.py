"""Config 2 device solve time (median of 7, L2 flushed) for the library named by
OTPRG_LIB; prints one line per seed.  Run twice with different OTPRG_LIB to A/B."""
import os, sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

lib = os.environ.get("OTPRG_LIB", "libotprg.so")
out = []
for seed in (1, 2, 3):
    S = otprg.Solver(0)
    S.prepare(otprg.gen_uniform_square(10000, seed), 0.01)
    ts = []
    for _ in range(7):
        S.flush_l2()
        m, s = S.solve_prepared()
        ts.append(s.device["solve_ms"])
    out.append(float(np.median(ts)))
    S.close()
print(f"{lib}: " + " ".join(f"{x:.3f}" for x in out) + f" mean {np.mean(out):.3f}", flush=True)
