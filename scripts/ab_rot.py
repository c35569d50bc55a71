"""Config 2 device solve time with the bench's access pattern: three prepared
instances (seeds 1/2/3, 600 MB of kT) solved round-robin without an L2 flush
(mean of 5 rounds after 2 warm-up rounds) for the library named by OTPRG_LIB."""
import os, sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

lib = os.environ.get("OTPRG_LIB", "libotprg.so")
S = [otprg.Solver(0) for _ in range(3)]
for k, seed in enumerate((1, 2, 3)):
    S[k].prepare(otprg.gen_uniform_square(10000, seed), 0.01)
ts = {1: [], 2: [], 3: []}
for r in range(7):
    for k, seed in enumerate((1, 2, 3)):
        m, s = S[k].solve_prepared()
        if r >= 2:
            ts[seed].append(s.device["solve_ms"])
out = [float(np.mean(ts[s])) for s in (1, 2, 3)]
print(f"{lib} (rotation): " + " ".join(f"{x:.3f}" for x in out) + f" mean {np.mean(out):.3f}", flush=True)
