"""Golden fixtures for config 3 (MNIST-shaped L1 costs) from the UNMODIFIED reference.

    make -C oracle && python tests/golden/make_golden_mnist.py

Writes the synthetic IDX3 file (paper_2203_03732_b200/instances.py, 20,000
images, generator seed 0) to a temporary path, then runs the reference's own
otpr::load_mnist_pair + otpr::solve_assignment (oracle/_ref) for each case and
stores the pins in tests/golden/mnist_pins.json (same hash definitions as
assign_pins.json).  The GPU tests regenerate the same file (it is
deterministic) instead of reading it from here.
"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Reference  # noqa: E402
from paper_2203_03732_b200.instances import make_synthetic_mnist  # noqa: E402

CASES = [(500, 1, (0.1, 0.05, 0.01, 0.2)), (1000, 1, (0.1, 0.05, 0.01)), (2000, 2, (0.1, 0.05, 0.01)),
         (10000, 1, (0.1, 0.05, 0.01))]


def main():
    ref = Reference.get()
    out = {}
    with tempfile.TemporaryDirectory() as d:
        path = make_synthetic_mnist(os.path.join(d, "synth-images-idx3-ubyte"), 20000, 0)
        for n, seed, epss in CASES:
            t0 = time.time()
            cost = ref.load_mnist_pair(path, n, seed)
            t_load = time.time() - t0
            for eps in epss:
                r = ref.solve_assignment(cost, eps, threads=1)
                key = f"mnist_n{n}_eps{eps!r}_s{seed}"
                out[key] = dict(kind="mnist", n_a=n, n_b=n, seed=seed, eps=eps, **r.pins(),
                                swapped=r.swapped, full_match_termination=r.full_match_termination,
                                ref_solve_ms=round(r.solve_ms, 3), ref_load_s=round(t_load, 2),
                                cost_min=float(cost.min()), cost_max=float(cost.max()))
                print(key, r.phases, f"load {t_load:.1f}s solve {r.solve_ms:.0f}ms", flush=True)
            del cost
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "mnist_pins.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
