"""Config 4 (n = 100k, eps = 0.01) sharded G = 1: precomputed kT slab vs on-the-fly costs."""
import sys, time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
inst = otprg.gen_uniform_square(n, 1)
res = {}
for otf in (False, True, False, True):
    t0 = time.perf_counter()
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01), 1, on_the_fly=otf)
    torch.cuda.synchronize()
    prep = (time.perf_counter() - t0) * 1e3
    ts = []
    for _ in range(3):
        sv.timer_start()
        m, s = sv.solve()
        ts.append(sv.timer_stop())
    key = (s.phases, s.sum_ni, int(np.sum(m.match_of_a.astype(np.int64) * np.arange(n) % 1000003)))
    print(f"on_the_fly={otf}: prepare {prep:.1f} ms, solve {[round(x, 2) for x in ts]} ms, {key}", flush=True)
    sv.close()
