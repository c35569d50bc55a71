import sys; sys.path.insert(0, ".")
import numpy as np, paper_2203_03732_b200 as otprg
rng = np.random.default_rng(7)
for n_a, n_b, levels in ((40, 900, 1), (600, 600, 2), (300, 700, 5), (257, 1000, 3)):
    mu = rng.integers(1, 50, n_a).astype(np.float64); nu = rng.integers(1, 50, n_b).astype(np.float64)
    mu /= mu.sum(); nu /= nu.sum()
    cost = rng.integers(0, levels, (n_a, n_b)) / max(1, levels - 1) if levels > 1 else np.full((n_a, n_b), 0.5)
    otprg.solve_ot(otprg.OTInstance(mu, nu, cost), 0.05)
