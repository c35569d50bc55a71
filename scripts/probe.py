"""Ad-hoc GPU probe: solve config-2 instances and print timings/pins."""
import json
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import pins_of  # noqa: E402

golden = json.load(open("tests/golden/assign_pins.json"))
solver = otprg.Solver(0)
for n, eps, seed in [(1000, 0.1, 1), (1000, 0.01, 1), (10000, 0.01, 1), (10000, 0.01, 2), (10000, 0.01, 3)]:
    inst = otprg.gen_uniform_square(n, seed)
    for storage in ("u8", "u16"):
        info = solver.prepare(inst, eps, storage)
        times = []
        for rep in range(4):
            solver.flush_l2()
            t0 = time.perf_counter()
            m, s = solver.solve_prepared()
            times.append((time.perf_counter() - t0) * 1e3)
        d = s.device
        key = f"square_n{n}_eps{eps!r}_s{seed}"
        p = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni, d["cost"])
        ok = all(p[k] == golden[key][k] for k in p) if key in golden else None
        print(f"{key} {storage}: parity={ok} phases={s.phases} build={info['build_ms']:.3f}ms "
              f"solve_dev={d['solve_ms']:.3f}ms phase1={d['phase1_ms']:.3f}ms wall={min(times):.3f}ms "
              f"touched={d['bytes_touched']/1e6:.1f}MB alg={d['bytes_alg']/1e6:.1f}MB", flush=True)
