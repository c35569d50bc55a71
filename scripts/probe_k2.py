"""K2 (points -> kT) build time: build_ms of prepare (events around the
range check + table + kernel), median of 5, n = 100k and 10k, u8 / u16."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

for n in (100_000, 10_000):
    inst = otprg.gen_uniform_square(n, 1)
    for storage in ("u8", "u16"):
        sv = otprg.Solver(0)
        ts = [sv.prepare(inst, 0.01, storage)["build_ms"] for _ in range(6)][1:]
        w = 1 if storage == "u8" else 2
        ms = float(np.median(ts))
        print(f"n={n} {storage}: build {ms:.3f} ms = {n * n * w / ms / 1e6:.0f} GB/s written", flush=True)
        sv.close()
