"""Golden pins for unbalanced instances at scale (SURVEY §8(f) rank 4:
orientation swap, assignment.cpp:385-399), from the UNMODIFIED reference.

Instance: the first n_a points of side A and the first n_b of side B of
otpr::gen_uniform_square(max(n_a, n_b), seed) (instances.cpp:48-78), cost
sqrt(dx^2+dy^2)/sqrt(2) as a dense matrix (bit-identical to the reference
formula).  Run in the build container: python tests/golden/make_golden_rect.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2203_03732_b200 as otprg  # noqa: E402  (host-side point streams only)
from oracle.pyoracle import Reference  # noqa: E402

CASES = [(4000, 2400, 21, 0.01), (2400, 4000, 22, 0.01), (16000, 10000, 31, 0.01),
         (10000, 16000, 32, 0.005)]


def main():
    ref = Reference.get()
    pins = {}
    for n_a, n_b, seed, eps in CASES:
        big = otprg.gen_uniform_square(max(n_a, n_b), seed)
        cost = otprg.points_cost(big.pts_a[:n_a], big.pts_b[:n_b])
        t0 = time.time()
        r = ref.solve_assignment(cost, eps, threads=1)
        key = f"rect_{n_a}x{n_b}_eps{eps!r}_s{seed}"
        pins[key] = dict(kind="rect_points", n_a=n_a, n_b=n_b, seed=seed, eps=eps, **r.pins(),
                         swapped=r.swapped, full_match_termination=r.full_match_termination)
        print(key, r.phases, f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "assign_rect_pins.json"), "w") as f:
        json.dump(pins, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
