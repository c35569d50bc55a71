"""Randomised OT parity sweep on the GPU against the UNMODIFIED reference
(oracle/_ref, built from /root/reference in the build container; the .so
travels with the repo): random masses (incl. zeros), shapes, eps; solve_ot
plans (entries, masses, cost bits, free_counts) and solve_copy_matching flows.
Usage: sweep_ot.py [seconds] [seed0]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2203_03732_b200 as otprg  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ref = Reference.get()
t_end = time.time() + budget
case = bad = 0
kinds = {}
while time.time() < t_end:
    case += 1
    seed = seed0 * 1_000_003 + case
    rng = np.random.default_rng(seed)
    kind = "ot" if rng.random() < 0.6 else "copy"
    big = rng.random() < 0.25  # (multi-block persistent loop, bucket merges)
    n_a, n_b = (int(rng.integers(100, 1500)), int(rng.integers(100, 1500))) if big else \
        (int(rng.integers(1, 120)), int(rng.integers(1, 120)))
    eps = float(np.exp(rng.uniform(np.log(0.02 if not big else 0.05), np.log(0.6))))
    fam = rng.random()
    if fam < 0.7:
        cost = rng.random((n_a, n_b))
    elif fam < 0.9:  # few levels: ties and runs of re-proposals in the claim rounds
        lv = int(rng.integers(2, 6))
        cost = rng.integers(0, lv, (n_a, n_b)) / (lv - 1)
    else:  # constant: every free b at the same cluster
        cost = np.full((n_a, n_b), float(rng.random()))
    if kind == "ot":
        w_a = rng.integers(0, 50, n_a).astype(np.float64)
        w_b = rng.integers(0, 50, n_b).astype(np.float64)
        w_a[0] += 1.0
        w_b[0] += 1.0
        mu, nu = w_a / w_a.sum(), w_b / w_b.sum()
        try:
            want = ref.solve_ot(mu, nu, cost, eps, entry_cap=(n_a + n_b) * 8 + 64)
        except Exception as e:  # noqa: BLE001
            print(f"case {case} seed {seed}: reference error {e}", flush=True)
            continue
        plan, st = otprg.solve_ot(otprg.OTInstance(mu, nu, cost), eps)
        ok = (plan.cost == want["cost"] and np.array_equal(plan.a, want["a"]) and np.array_equal(plan.b, want["b"])
              and plan.mass.tobytes() == want["mass"].tobytes() and np.array_equal(st.free_counts, want["free_counts"]))
        tag = f"ot {n_a}x{n_b} eps={eps:.3g}"
    else:
        k, uf, uc = ref.scale_round_costs(cost, eps)
        d = rng.integers(0, 15, n_a).astype(np.int64)
        d[0] += 1
        s, tot = [], 0
        for _ in range(n_b):
            room = int(d.sum()) - tot
            c = int(rng.integers(0, room + 1)) if room > 0 else 0
            s.append(c)
            tot += c
        s = np.array(s, np.int64)
        want = ref.solve_copy_matching(k, eps, uf, uc, d, s, eps, check=True, phase_cap=1)
        chk = bool(rng.random() < 0.5)  # (without the checks: the persistent phase loop)
        res = otprg.solve_copy_matching(otprg.CopyInstance(otprg.ScaledCosts(eps, k, uf, uc), d, s), eps,
                                        otprg.ClusterOptions(check_invariants=chk))
        ok = (np.array_equal(res.flow, want["flow"]) and res.stats.phases == want["phases"]
              and np.array_equal(res.stats.free_counts, want["free_counts"]))
        tag = f"copy {n_a}x{n_b} eps={eps:.3g} copies {int(d.sum())}/{int(s.sum())}"
    kinds[kind] = kinds.get(kind, 0) + 1
    if not ok:
        bad += 1
        print(f"MISMATCH case {case} seed {seed}: {tag}", flush=True)
print(f"cases {case} mismatches {bad} by kind {kinds}", flush=True)
