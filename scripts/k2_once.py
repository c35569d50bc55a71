"""One K2 build (gen_uniform_square(n, 1) -> kT, eps 0.01) — a short command for ncu."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
storage = sys.argv[2] if len(sys.argv) > 2 else "u16"
sv = otprg.Solver(0)
print(sv.prepare(otprg.gen_uniform_square(n, 1), 0.01, storage)["build_ms"])
