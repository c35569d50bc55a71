"""One on-the-fly sharded (G = 1) config-4 solve: a short command for ncu."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

sv = ShardedSolver(otprg.gen_uniform_square(100_000, 1), otprg.AssignmentOptions(eps=0.01), 1, on_the_fly=True)
m, s = sv.solve()
print("phases", s.phases, "refills", s.device["refill_rounds"])
