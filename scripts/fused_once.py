"""One fused single-GPU solve of gen_uniform_square(n, 1) (for ncu): python scripts/fused_once.py n eps storage"""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
storage = sys.argv[3] if len(sys.argv) > 3 else "u16"
sv = otprg.Solver(0)
sv.prepare(otprg.gen_uniform_square(n, 1), eps, storage)
m, s = sv.solve_prepared()
print("phases", s.phases, "solve_ms", s.device["solve_ms"])
