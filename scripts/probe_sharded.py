"""Time the sharded path with G logical shards on one GPU (per-phase protocol
cost) against the fused single-GPU solver.  Usage: probe_sharded.py N [K]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
eps = 0.01
inst = otprg.gen_uniform_square(n, 1)
opt = otprg.AssignmentOptions(eps=eps, storage="u16")
sv1 = otprg.Solver(0)
m1, s1 = sv1.solve(inst, opt)
print(f"fused: phases {s1.phases} sum_ni {s1.sum_ni} solve_ms {s1.device['solve_ms']:.3f} "
      f"build_ms {s1.device['build_ms']:.3f}", flush=True)
sv1.close()
for G in (1, 2, 4, 8):
    t0 = time.perf_counter()
    sv = ShardedSolver(inst, opt, G, K=K)
    prep = time.perf_counter() - t0
    m, s = sv.solve()
    same = (np.array_equal(m.match_of_a, m1.match_of_a)
            and np.array_equal(s.duals_final.y_a, s1.duals_final.y_a)
            and np.array_equal(s.duals_final.y_b, s1.duals_final.y_b))
    ts = []
    for _ in range(3):
        sv.timer_start()
        sv.solve()
        ts.append(sv.timer_stop())
    sv.close()
    print(f"G={G} K={K}: same={same} phases {s.phases} rounds {s.device['refill_rounds']} "
          f"ms {np.mean(ts):.3f} (per phase {np.mean(ts) / max(1, s.phases):.3f}) prep {prep:.2f}s",
          flush=True)
