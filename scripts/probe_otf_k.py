"""Config 4 sharded on-the-fly: solve time vs the candidate count K."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

inst = otprg.gen_uniform_square(100_000, 1)
for otf in (True, False):
    for K in (2, 4, 8, 16, 32):
        sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01), 1, K=K, on_the_fly=otf)
        ts = []
        for _ in range(3):
            sv.timer_start()
            m, s = sv.solve()
            ts.append(sv.timer_stop())
        print(f"otf={otf} K={K}: solve {min(ts):.2f} ms refills {s.device['refill_rounds']} phases {s.phases}", flush=True)
        sv.close()
