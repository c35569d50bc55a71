"""One config-2 solve (seed 1) through the C ABI: a short command for ncu."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

storage = sys.argv[1] if len(sys.argv) > 1 else "u16"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(10000, 1), 0.01, storage)
for _ in range(reps):
    m, s = S.solve_prepared()
    print("phases", s.phases, "solve_ms", s.device["solve_ms"], "phase1_ms", s.device["phase1_ms"],
          flush=True)
