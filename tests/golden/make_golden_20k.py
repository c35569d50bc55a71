"""Golden fixtures for config 4's code paths at the largest size the
reference runs here ("pin n <= 20k runs of the same code path
against the oracle").

    make -C oracle ref && python tests/golden/make_golden_20k.py

Runs the UNMODIFIED reference (oracle/_ref/libotpr_ref.so, threads = 1) on
otpr::gen_uniform_square(20000, seed) (instances.cpp:48-78) at eps = 0.01 —
about 1-2 minutes and 4.8 GB of host memory per seed — and writes
tests/golden/assign20k_pins.json plus the full outputs
tests/golden/assign_square_n20000_eps0.01_s<seed>.npz.  The GPU tests pin
the fused, sharded (G = 1/2/4/8, K = 1/16) and on-the-fly solvers to them.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [(20000, 0.01, 1), (20000, 0.01, 2)]


def main() -> None:
    ref = Reference.get()
    pins = {}
    for n, eps, seed in CASES:
        t0 = time.time()
        key = f"square_n{n}_eps{eps!r}_s{seed}"
        r = ref.solve_uniform_square(n, seed, eps, threads=1)
        pins[key] = dict(kind="square", n_a=n, n_b=n, seed=seed, eps=eps, **r.pins(),
                         swapped=r.swapped, full_match_termination=r.full_match_termination,
                         ref_solve_ms=round(r.solve_ms, 3))
        np.savez_compressed(os.path.join(OUT, f"assign_{key}.npz"), match_of_a=r.match_of_a,
                            y_a=r.y_a.astype(np.int16), y_b=r.y_b.astype(np.int16),
                            free_counts=r.free_counts.astype(np.int32))
        print(key, pins[key]["phases"], pins[key]["sum_ni"], f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(OUT, "assign20k_pins.json"), "w") as f:
        json.dump(pins, f, indent=1, sort_keys=True)
    print("wrote", len(pins), "cases")


if __name__ == "__main__":
    main()
