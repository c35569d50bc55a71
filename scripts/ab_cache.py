"""A/B of the phase-loop shared-memory row cache (OTPRG_ROW_CACHE=0 disables):
config 2 (n = 10k, eps = 0.01) seeds 1-3, device solve ms (median of 5) and pins."""
import os, sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
storage = sys.argv[3] if len(sys.argv) > 3 else "auto"
for seed in (1, 2, 3):
    inst = otprg.gen_uniform_square(n, seed)
    res = {}
    for mode in ("0", "on", "0", "on"):
        if mode == "0":
            os.environ["OTPRG_ROW_CACHE"] = "0"
        else:
            os.environ.pop("OTPRG_ROW_CACHE", None)
        S = otprg.Solver(0)
        S.prepare(inst, eps, storage)
        ts = []
        for _ in range(5):
            S.flush_l2()
            m, s = S.solve_prepared()
            ts.append(s.device["solve_ms"])
        key = (s.phases, s.sum_ni, int(np.sum(m.match_of_a.astype(np.int64) * np.arange(n) % 1000003)))
        res.setdefault(mode, []).append((float(np.median(ts)), key))
        S.close()
    k0 = {r[1] for r in res["0"]}
    k1 = {r[1] for r in res["on"]}
    print(f"seed {seed}: off {[round(r[0], 3) for r in res['0']]} on {[round(r[0], 3) for r in res['on']]} "
          f"same={k0 == k1 and len(k0) == 1} {k0}", flush=True)
