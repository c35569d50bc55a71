"""A/B of the idle-warp cache prebuild: config 2 device solve (kT resident,
L2 flushed), median of 7 per seed; run with OTPRG_PREBUILD=0 and without."""
import os, sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

tag = os.environ.get("OTPRG_PREBUILD", "1")
out = []
for seed in (1, 2, 3):
    S = otprg.Solver(0)
    S.prepare(otprg.gen_uniform_square(10000, seed), 0.01, sys.argv[1] if len(sys.argv) > 1 else "u16")
    ts = []
    for _ in range(7):
        S.flush_l2()
        m, s = S.solve_prepared()
        ts.append(s.device["solve_ms"])
    out.append(float(np.median(ts)))
    st = s.device["chain_stats"]
    S.close()
print(f"prebuild={tag}: " + " ".join(f"{x:.3f}" for x in out) + f" mean {np.mean(out):.3f}  (seed 3 chains: rescan {st['rescan']} cache_hit {st['cache_hit']})", flush=True)
