"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

It calls oracle/_ref/libotpr_ref.so (reference sources compiled by
oracle/Makefile) through oracle/pyoracle.py and writes

* tests/golden/assign_pins.json  — per case: phases, sum_ni, swapped,
  full_match_termination, cost (hex), FNV-1a-64 of match_of_a (int32 LE),
  y_a||y_b (int64 LE) and free_counts (int64 LE);
* tests/golden/assign_<case>.npz — full outputs for first-divergence debugging.

Instances:
* ``square``: otpr::gen_uniform_square(n, seed) (instances.cpp:48-78);
* ``random``: test_util.hpp:19-30 random_instance (row-major u01 draws from
  std::mt19937_64(seed)), regenerated in the tests from the same stream.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SQUARE = (
    [(1000, 0.1, s) for s in range(1, 31)]
    + [(1000, 0.01, s) for s in (1, 2, 3)]
    + [(1000, e, 1) for e in (0.05, 0.02, 1.0 / 300.0, 0.125, 0.07, 0.2)]
    + [(2000, 0.01, 3), (3000, 0.02, 1), (4000, 0.1, 1), (4000, 0.01, 1)]
    + [(10000, 0.01, s) for s in (1, 2, 3)]
    + [(10000, 0.1, 1), (10000, 0.05, 1)]
)
RANDOM = [
    (50, 50, s, e) for s in range(1, 6) for e in (0.1, 0.05)
] + [
    (12, 5, 77, 0.1), (5, 12, 78, 0.1), (60, 60, 1234, 0.1), (10, 10, 2024, 0.99),
    (40, 40, 555, 0.08), (9, 7, 21, 0.07), (200, 130, 7, 0.03), (130, 200, 8, 0.03),
    (300, 300, 9, 0.01), (1, 1, 3, 0.5),
] + [(30, 30, s * 131, 0.15 if s % 2 == 0 else 0.08) for s in range(1, 9)]


def random_instance(n_a: int, n_b: int, seed: int) -> np.ndarray:
    """test_util.hpp:19-30: row-major u01 from mt19937_64(seed)."""
    raw = Oracle.get().raw_stream(seed, n_a * n_b)
    return ((raw >> np.uint64(11)).astype(np.float64) * 2.0**-53).reshape(n_a, n_b)


def main() -> None:
    ref = Reference.get()
    pins = {}
    t0 = time.time()
    for n, eps, seed in SQUARE:
        key = f"square_n{n}_eps{eps!r}_s{seed}"
        r = ref.solve_uniform_square(n, seed, eps, threads=1)
        pins[key] = dict(kind="square", n_a=n, n_b=n, seed=seed, eps=eps, **r.pins(),
                         swapped=r.swapped, full_match_termination=r.full_match_termination,
                         ref_solve_ms=round(r.solve_ms, 3))
        np.savez_compressed(os.path.join(OUT, f"assign_{key}.npz"), match_of_a=r.match_of_a,
                            y_a=r.y_a.astype(np.int16), y_b=r.y_b.astype(np.int16),
                            free_counts=r.free_counts.astype(np.int32))
        print(key, pins[key]["phases"], f"{time.time() - t0:.1f}s", flush=True)
    for n_a, n_b, seed, eps in RANDOM:
        key = f"random_{n_a}x{n_b}_eps{eps!r}_s{seed}"
        cost = random_instance(n_a, n_b, seed)
        r = ref.solve_assignment(cost, eps, threads=1)
        pins[key] = dict(kind="random", n_a=n_a, n_b=n_b, seed=seed, eps=eps, **r.pins(),
                         swapped=r.swapped, full_match_termination=r.full_match_termination)
        np.savez_compressed(os.path.join(OUT, f"assign_{key}.npz"), match_of_a=r.match_of_a,
                            y_a=r.y_a, y_b=r.y_b, free_counts=r.free_counts)
    with open(os.path.join(OUT, "assign_pins.json"), "w") as f:
        json.dump(pins, f, indent=1, sort_keys=True)
    print("wrote", len(pins), "cases")


if __name__ == "__main__":
    main()
