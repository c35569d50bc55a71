"""Config 4 sharded G=1 (u8 slab, resident loop): solve time vs K."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

inst = otprg.gen_uniform_square(100_000, 1)
for K in (8, 16, 24, 32):
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01, storage="u8"), 1, K=K)
    ts = []
    for _ in range(5):
        sv.timer_start()
        m, s = sv.solve()
        ts.append(sv.timer_stop())
    print(f"K={K}: {np.median(ts):.3f} ms, refills {s.device['refill_rounds']}, phases {s.phases}", flush=True)
    sv.close()
