"""Config-3 cost build (K3: L1/2 of normalised 784-pixel images + rounding)
at n = 10k, timed over repeats; a short command for ncu of l1_round_kernel."""
import os
import sys
import tempfile
import time
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.instances import make_synthetic_mnist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
path = make_synthetic_mnist(os.path.join(tempfile.mkdtemp(), "synth-idx3"), 2 * n, 0)
inst = otprg.load_mnist_pair(path, n, 1)
S = otprg.Solver(0)
ts = []
for _ in range(reps):
    t = time.perf_counter()
    S.prepare(inst, 0.01)
    ts.append((time.perf_counter() - t) * 1e3)
print("prepare ms", " ".join(f"{x:.2f}" for x in ts))
