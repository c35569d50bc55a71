"""Fused single-GPU solve at n = 100k (config 4): chain statistics."""
import sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(100_000, 1), 0.01)
for _ in range(2):
    m, s = S.solve_prepared()
print("solve_ms", round(s.device["solve_ms"], 3), "phases", s.phases, "sum_ni", s.sum_ni)
print("chain stats", s.device["chain_stats"], "bytes_touched MB", s.device["bytes_touched"] / 1e6)
print("free_counts head", list(s.free_counts[:12]), "tail", list(s.free_counts[-5:]))
