"""Repro: fused u32 solve of a rectangular point instance (sanitizer target)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2203_03732_b200 as otprg

rng = np.random.default_rng(17)
for storage in ("u8", "u16", "u32"):
    rng = np.random.default_rng(17)
    for n_a, n_b, eps in ((2500, 1300, 0.02), (900, 2100, 0.05), (64, 64, 0.003)):
        inst = otprg.AssignmentInstance(n_a, n_b, pts_a=rng.random((n_a, 2)), pts_b=rng.random((n_b, 2)))
        opt = otprg.AssignmentOptions(eps=eps, storage=storage)
        sv = otprg.Solver(0)
        try:
            m, s = sv.solve(inst, opt)
        except otprg.ParameterError as e:
            print(storage, n_a, n_b, eps, "ParameterError", e, flush=True)
            sv.close()
            continue
        print(storage, n_a, n_b, eps, s.phases, flush=True)
        sv.close()
