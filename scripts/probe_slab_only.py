"""Config 4 sharded G = 1 with the precomputed slab: best of 3 device solve times."""
import os, sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

sv = ShardedSolver(otprg.gen_uniform_square(100_000, 1), otprg.AssignmentOptions(eps=0.01), 1, on_the_fly=False)
ts = []
for _ in range(4):
    sv.timer_start()
    m, s = sv.solve()
    ts.append(sv.timer_stop())
print(f"{os.environ.get('OTPRG_LIB', 'libotprg.so')}: slab solve best {min(ts):.2f} ms phases {s.phases}", flush=True)
