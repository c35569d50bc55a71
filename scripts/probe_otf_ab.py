"""Config 4 sharded G = 1 on the fly (u8 and u16 t), best of 4 device solve times, for OTPRG_LIB."""
import os, sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

inst = otprg.gen_uniform_square(100_000, 1)
for storage in ("u8", "u16"):
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01, storage=storage), 1, on_the_fly=True)
    ts = []
    for _ in range(4):
        sv.timer_start()
        m, s = sv.solve()
        ts.append(sv.timer_stop())
    sv.close()
    print(f"{os.environ.get('OTPRG_LIB', 'libotprg.so')} {storage}: otf solve best {min(ts):.2f} ms "
          f"phases {s.phases}", flush=True)
