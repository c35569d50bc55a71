"""One sharded config-4 solve (a short command for ncu):
python scripts/sharded_once.py G n storage otf(0/1) resident(0/1)"""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

a = sys.argv[1:] + [None] * 5
G = int(a[0] or 1)
n = int(a[1] or 100_000)
storage = a[2] or "u16"
otf = bool(int(a[3] or 0))
resident = bool(int(a[4] or 1))
sv = ShardedSolver(otprg.gen_uniform_square(n, 1), otprg.AssignmentOptions(eps=0.01, storage=storage), G,
                   on_the_fly=otf, resident=resident)
m, s = sv.solve()
print("phases", s.phases, "refills", s.device["refill_rounds"], "solve_ms", s.device["solve_ms"])
