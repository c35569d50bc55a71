"""Config 4 sharded G = 1 (u8 slab, u16 slab, u8 on the fly), best of 4 device solve times, for OTPRG_LIB."""
import os, sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

inst = otprg.gen_uniform_square(100_000, 1)
out = []
for storage, otf in (("u8", False), ("u16", False), ("u8", True)):
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01, storage=storage), 1, on_the_fly=otf)
    ts = []
    for _ in range(4):
        sv.timer_start()
        m, s = sv.solve()
        ts.append(sv.timer_stop())
    sv.close()
    out.append(f"{storage}{'-otf' if otf else ''} {min(ts):.2f}")
print(os.environ.get("OTPRG_LIB", "libotprg.so"), " | ".join(out), flush=True)
