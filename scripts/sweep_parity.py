"""Randomised parity sweep on the GPU: random shapes, eps, cost families and
storage widths (plus the sharded path with random shard counts / K) against
the C oracle, for a wall-clock budget.  Prints every mismatch with the seed
that reproduces it.  Usage: sweep_parity.py [seconds] [seed0]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2203_03732_b200 as otprg  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402
from paper_2203_03732_b200 import sharded  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
verbose = len(sys.argv) > 3 and sys.argv[3] == "-v"
orc = Oracle.get()
t_end = time.time() + budget
case = 0
bad = 0
counts = {}


def family_cost(rng, n_a, n_b, fam):
    if fam == "uniform":
        return rng.random((n_a, n_b))
    if fam == "levels":  # few distinct values: many ties
        return rng.integers(0, 5, (n_a, n_b)) / 4.0
    if fam == "lowrank":  # c = |x_a - y_b| on a line: structured ties
        x, y = rng.random(n_a), rng.random(n_b)
        return np.abs(x[:, None] - y[None, :])
    if fam == "tiny":  # near-zero costs with rare large ones
        c = rng.random((n_a, n_b)) * 0.02
        c[rng.random((n_a, n_b)) < 0.05] = 1.0
        return c
    raise ValueError(fam)


only = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else None
while time.time() < t_end:
    case += 1
    if only is not None:
        if not only:
            break
        case = only.pop(0)
    seed = seed0 * 1_000_003 + case
    rng = np.random.default_rng(seed)
    if verbose:
        print(f"start case {case} seed {seed}", flush=True)
    if case % 1000 == 0:
        import torch
        print(f"case {case}: free device memory {torch.cuda.mem_get_info(0)[0] / 2**30:.2f} GiB", flush=True)
    kind = rng.choice(["dense", "dense", "dense", "points", "sharded", "otf"])
    if kind == "dense":
        n_a, n_b = int(rng.integers(1, 1500)), int(rng.integers(1, 1500))
        fam = str(rng.choice(["uniform", "levels", "lowrank", "tiny"]))
        eps = float(np.exp(rng.uniform(np.log(0.004), np.log(0.6))))
        if rng.random() < 0.05 and n_a * n_b <= 400:
            eps = float(np.exp(rng.uniform(np.log(2e-6), np.log(2e-5))))  # uint32 storage
        cost = family_cost(rng, n_a, n_b, fam)
        inst = otprg.AssignmentInstance(n_a, n_b, cost)
        storage = str(rng.choice(["auto", "u8", "u16", "u32"]))
        try:
            want = orc.solve_assignment(cost, eps)
        except Exception as e:  # noqa: BLE001
            print(f"case {case} seed {seed}: oracle error {e}", flush=True)
            continue
        try:
            m, s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps, storage=storage))
        except otprg.ParameterError:
            continue  # storage too narrow for this eps
        ok = (np.array_equal(m.match_of_a, want.match_of_a) and np.array_equal(s.duals_final.y_a, want.y_a)
              and np.array_equal(s.duals_final.y_b, want.y_b) and s.phases == want.phases
              and np.array_equal(s.free_counts, want.free_counts) and s.device["cost"] == want.cost)
        tag = f"dense {n_a}x{n_b} {fam} eps={eps:.3g} {storage}"
    else:
        n = int(rng.integers(2, 2500))
        n_b = n if rng.random() < 0.6 else int(rng.integers(2, 2500))
        eps = float(np.exp(rng.uniform(np.log(0.005), np.log(0.3))))
        pa, pb = rng.random((n, 2)), rng.random((n_b, 2))
        inst = otprg.AssignmentInstance(n, n_b, pts_a=pa, pts_b=pb)
        cost = otprg.points_cost(pa, pb) if hasattr(otprg, "points_cost") else None
        ref_m, ref_s = otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps))
        if kind == "points":
            want = orc.solve_assignment(np.ascontiguousarray(cost), eps)
            ok = (np.array_equal(ref_m.match_of_a, want.match_of_a) and ref_s.phases == want.phases
                  and np.array_equal(ref_s.duals_final.y_b, want.y_b) and ref_s.device["cost"] == want.cost)
            tag = f"points {n}x{n_b} eps={eps:.3g}"
        else:
            G, K = int(rng.integers(1 if kind == "otf" else 2, 6)), int(rng.choice([1, 2, 4, 16]))
            m2, s2 = sharded.solve_assignment_sharded(inst, otprg.AssignmentOptions(eps=eps), G, K=K,
                                                      on_the_fly=kind == "otf")
            ok = (np.array_equal(ref_m.match_of_a, m2.match_of_a) and s2.phases == ref_s.phases
                  and np.array_equal(ref_s.duals_final.y_a, s2.duals_final.y_a)
                  and np.array_equal(ref_s.duals_final.y_b, s2.duals_final.y_b))
            tag = f"{kind} {n}x{n_b} eps={eps:.3g} G={G} K={K}"
    counts[kind] = counts.get(kind, 0) + 1
    if verbose:
        print(f"ok case {case} seed {seed}: {tag}", flush=True)
    if not ok:
        bad += 1
        print(f"MISMATCH case {case} seed {seed}: {tag}", flush=True)
print(f"cases {case} mismatches {bad} by kind {counts}", flush=True)
