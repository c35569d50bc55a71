"""Golden fixtures for the OT path (config 5) from the UNMODIFIED reference.

    make -C oracle && python tests/golden/make_golden_ot.py [--micro-only]

Cases: the micro instances of tests/test_ot.cpp and
otpr::gen_random_ot_rational(n_a, n_b, seed) (instances.cpp:159-191) solved
by otpr::solve_ot(eps) (ot.cpp:705-732) through oracle/_ref.  Stores
tests/golden/ot_pins.json (phases, sum_ni, theta, copy totals, plan size and
cost bits, FNV-1a-64 of the plan arrays) and full plans for small cases.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference, fnv1a64  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MICRO = {
    "micro_1x1": ([1.0], [1.0], [[0.2]], 0.1),
    "micro_antidiag": ([0.5, 0.5], [0.5, 0.5], [[0.0, 1.0], [1.0, 0.0]], 0.1),
    "micro_2x2_theta": ([0.55, 0.45], [0.3, 0.7], [[0.1, 0.2], [0.3, 0.4]], 0.5),
    "micro_dyadic": ([0.25, 0.75], [0.5, 0.5], [[0.1, 0.2], [0.3, 0.4]], 0.5),
}
# eps below ~4.58e-5 (eps/3 below 1/65531): the device stores k as uint32
MICRO.update({f"{k}_eps4.5e-5": (mu, nu, c, 4.5e-5) for k, (mu, nu, c, _) in list(MICRO.items())})
RATIONAL = ([(10, 10, s * 7, e) for s in range(1, 6) for e in (0.25, 0.1)]
            + [(6, 4, 3, 0.23), (50, 50, 1, 0.1), (100, 100, 1, 0.1), (100, 100, 1, 0.01),
               (300, 200, 3, 0.05), (200, 300, 4, 0.05), (1000, 1000, 1, 0.01), (1000, 1000, 2, 0.05),
               (5000, 5000, 1, 0.01), (20000, 20000, 1, 0.01)])


def pins(r):
    return {"phases": int(r["phases"]), "sum_ni": int(r["sum_ni"]), "cost_hex": float(r["cost"]).hex(),
            "theta_hex": float(r["theta"]).hex(), "total_d": int(r["total_d"]),
            "total_s": int(r["total_s"]), "n_entries": int(r["n_entries"]),
            "fnv_a": "%016x" % fnv1a64(r["a"].astype(np.int32)),
            "fnv_b": "%016x" % fnv1a64(r["b"].astype(np.int32)),
            "fnv_mass": "%016x" % fnv1a64(r["mass"].astype(np.float64)),
            "fnv_free": "%016x" % fnv1a64(r["free_counts"].astype(np.int64))}


def main(micro_only=False):
    """micro_only: regenerate the micro cases into the existing ot_pins.json."""
    ref = Reference.get()
    out = {}
    if micro_only:
        with open(os.path.join(OUT, "ot_pins.json")) as f:
            out = {k: v for k, v in json.load(f).items() if v["kind"] != "micro"}
    for key, (mu, nu, cost, eps) in MICRO.items():
        r = ref.solve_ot(mu, nu, np.array(cost), eps)
        out[key] = dict(kind="micro", mu=mu, nu=nu, cost=cost, eps=eps, **pins(r))
        np.savez_compressed(os.path.join(OUT, f"ot_{key}.npz"), a=r["a"], b=r["b"], mass=r["mass"],
                            free_counts=r["free_counts"])
    for n_a, n_b, seed, eps in ([] if micro_only else RATIONAL):
        key = f"ot_rational_{n_a}x{n_b}_s{seed}_eps{eps!r}"
        t0 = time.time()
        r = ref.solve_ot_rational(n_a, n_b, seed, eps, entry_cap=(n_a + n_b) * 8 + 64)
        out[key] = dict(kind="rational", n_a=n_a, n_b=n_b, seed=seed, eps=eps, **pins(r),
                        ref_solve_ms=round(r["solve_ms"], 2))
        if n_a * n_b <= 1_000_000:
            np.savez_compressed(os.path.join(OUT, f"ot_{key}.npz"), a=r["a"], b=r["b"], mass=r["mass"],
                                free_counts=r["free_counts"])
        print(key, r["phases"], r["n_entries"], f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(OUT, "ot_pins.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(micro_only="--micro-only" in sys.argv)
