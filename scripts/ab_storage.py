"""Config 2 device solve time per cost-storage width (median of 7, L2 flushed):
u8 (100 MB kT, fits the 126 MB L2) vs u16 (200 MB) vs u32."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

for storage in ("u8", "u16", "u32"):
    out = []
    for seed in (1, 2, 3):
        S = otprg.Solver(0)
        S.prepare(otprg.gen_uniform_square(10000, seed), 0.01, storage)
        ts = []
        for _ in range(7):
            S.flush_l2()
            m, s = S.solve_prepared()
            ts.append(s.device["solve_ms"])
        out.append(float(np.median(ts)))
        S.close()
    print(f"{storage}: " + " ".join(f"{x:.3f}" for x in out) + f" mean {np.mean(out):.3f}", flush=True)
