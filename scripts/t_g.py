import sys; sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg
from paper_2203_03732_b200 import sharded
n = int(sys.argv[1]); G = int(sys.argv[2]); res = sys.argv[3] == "1"
inst = otprg.gen_uniform_square(n, 3)
m, s = sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=0.01), G, resident=res)
print("ok", n, G, res, s.phases, flush=True)
