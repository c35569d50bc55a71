"""Golden fixtures for the copy/cluster solver (otpr::solve_copy_matching,
ot.cpp:418-637) and its checks, from the UNMODIFIED reference via oracle/_ref.

    make -C oracle ref && python tests/golden/make_golden_copy.py

Copy instances are drawn like tests/test_ot.cpp:234-346 (a micro grid and
"larger instances") plus a few wider ones: u01 costs rounded by the
reference's scale_round_costs at eps, copy counts with total supply <= total
demand.  Stored per group in tests/golden/copy_<group>.npz under keys
"<case>_<field>": the instance (k, unit_floor/ceil, copies, eps), the final
flow (completion included), free_counts, phases / sum_ni / full-match flag,
the flow matrix and n_i after every phase (observer; first 64 phases) and
the final ClusterState in the flat layout of include/otprg.h.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import FLAT_KEYS, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GROUPS = {  # name: (seed, cases, max vertices, max copies, eps choices, max copy total)
    "micro": (2024, 15, 3, 3, (0.2, 0.3, 0.4, 0.5), 12),
    "larger": (777, 25, 5, 12, (0.1, 0.15, 0.2, 0.25, 0.3), None),
    "wide": (4242, 6, 60, 40, (0.05, 0.1), None),
}


def cases(seed, count, max_v, max_c, eps_choices, max_total):
    rng = np.random.default_rng(seed)
    while count > 0:
        eps = float(rng.choice(eps_choices))
        lo = 1 if max_v <= 5 else max_v // 3
        n_a, n_b = int(rng.integers(lo, max_v + 1)), int(rng.integers(lo, max_v + 1))
        d = rng.integers(1, max_c + 1, n_a).astype(np.int64)
        s, total = [], 0
        for _ in range(n_b):
            room = int(d.sum()) - total
            c = int(rng.integers(0, room + 1)) if room > 0 else 0
            s.append(c)
            total += c
        s = np.array(s, np.int64)
        if total == 0 or (max_total and int(d.sum()) + total > max_total):
            continue
        count -= 1
        yield rng.random((n_a, n_b)), d, s, eps


def main():
    ref = Reference.get()
    for group, (seed, count, max_v, max_c, eps_choices, max_total) in GROUPS.items():
        out = {}
        for i, (cost, d, s, eps) in enumerate(cases(seed, count, max_v, max_c, eps_choices, max_total)):
            k, uf, uc = ref.scale_round_costs(cost, eps)
            r = ref.solve_copy_matching(k, eps, uf, uc, d, s, eps, check=True, phase_cap=64)
            rec = dict(k=k, unit_floor=uf, unit_ceil=uc, demand_copies=d, supply_copies=s, eps=eps,
                       flow=r["flow"], free_counts=r["free_counts"], phases=r["phases"], sum_ni=r["sum_ni"],
                       full_match_termination=int(r["full_match_termination"]),
                       phase_flows=r["phase_flows"], phase_ni=r["phase_ni"],
                       **{f"state_{x}": r["state"][x] for x in FLAT_KEYS})
            out.update({f"{i}_{key}": np.asarray(v) for key, v in rec.items()})
            print(group, i, k.shape, int(d.sum()), int(s.sum()), eps, r["phases"], flush=True)
        np.savez_compressed(os.path.join(OUT, f"copy_{group}.npz"), **out)


if __name__ == "__main__":
    main()
