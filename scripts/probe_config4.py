"""Config 4 (n = 100k, eps = 0.01) on one GPU: fused solver vs sharded G = 1
(resident graph loop and host-driven), slab u8 / u16 and on the fly.
Median of 5 device-timed solves each (CUDA events on the solver's stream)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

inst = otprg.gen_uniform_square(100_000, 1)
ref = None
for storage in ("u16", "u8"):
    sv = otprg.Solver(0)
    info = sv.prepare(inst, 0.01, storage)
    ts = []
    for _ in range(5):
        sv.timer_start()
        m, s = sv.solve_prepared()
        ts.append(sv.timer_stop())
    if ref is None:
        ref = (m, s)
    print(f"fused {storage}: build {info['build_ms']:.2f} ms, solve {np.median(ts):.3f} ms, phases {s.phases}", flush=True)
    sv.close()
for storage, otf, resident in (("u16", False, True), ("u8", False, True), ("u16", True, True),
                               ("u8", True, True), ("u16", False, False), ("u16", True, False)):
    t0 = time.perf_counter()
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01, storage=storage), 1, K=16, on_the_fly=otf,
                       resident=resident)
    prep = time.perf_counter() - t0
    ts = []
    for _ in range(5):
        sv.timer_start()
        m, s = sv.solve()
        ts.append(sv.timer_stop())
    same = (np.array_equal(m.match_of_a, ref[0].match_of_a) and np.array_equal(s.duals_final.y_b, ref[1].duals_final.y_b)
            and s.phases == ref[1].phases)
    print(f"sharded G=1 {storage} otf={otf} resident={resident}: prep {prep*1e3:.1f} ms, solve {np.median(ts):.3f} ms "
          f"(min {min(ts):.3f}), refills {s.device['refill_rounds']}, launches {s.device['gpu_launches']}, "
          f"identical {same}", flush=True)
    sv.close()
