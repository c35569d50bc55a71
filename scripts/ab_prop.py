"""Phase-1 propose scan A/B for OTPRG_LIB: median %globaltimer span
(phase1_ms) of config 2 (kT resident), (a) seed 1 with an L2 flush before
every solve, (b) seeds 1/2/3 rotating without a flush (the bench's form)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

lib = os.environ.get("OTPRG_LIB", "libotprg.so")
res = []
for storage in ("u16", "u8"):
    S = [otprg.Solver(0) for _ in range(3)]
    for i, sv in enumerate(S):
        sv.prepare(otprg.gen_uniform_square(10000, i + 1), 0.01, storage)
    fl, rot = [], []
    for _ in range(15):
        S[0].flush_l2()
        fl.append(S[0].solve_prepared()[1].device["phase1_ms"])
    for k in range(30):
        rot.append(S[k % 3].solve_prepared()[1].device["phase1_ms"])
    w = 1 if storage == "u8" else 2
    B = 10000 * 10000 * w
    res.append(f"{storage}: flush {np.median(fl)*1e3:.1f} us ({B/np.median(fl)/1e6:.0f} GB/s) "
               f"rotate {np.median(rot)*1e3:.1f} us ({B/np.median(rot)/1e6:.0f} GB/s)")
    for sv in S:
        sv.close()
print(f"{lib}: " + " | ".join(res), flush=True)
