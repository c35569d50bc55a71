"""Solve time of config 2 (seeds 1-3, u8/u16) for the library in $OTPRG_LIB."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

out = []
for storage in ("u8", "u16"):
    ms, p1 = [], []
    for seed in (1, 2, 3):
        S = otprg.Solver(0)
        S.prepare(otprg.gen_uniform_square(10000, seed), 0.01, storage)
        best = 1e9
        for _ in range(3):
            S.flush_l2()
            m, s = S.solve_prepared()
            best = min(best, s.device["solve_ms"])
        ms.append(best)
        p1.append(s.device["phase1_ms"])
        S.close()
    out.append(f"{storage}: seeds {['%.3f' % x for x in ms]} mean {np.mean(ms):.3f} ms phase1 {np.mean(p1)*1e3:.0f} us")
print(os.environ.get("OTPRG_LIB", "libotprg.so"), " | ".join(out), flush=True)
