"""One sharded (G logical shards) config-4 solve: a short command for ncu."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
sv = ShardedSolver(otprg.gen_uniform_square(n, 1), otprg.AssignmentOptions(eps=0.01), G)
m, s = sv.solve()
print("phases", s.phases, "refills", s.device["refill_rounds"])
