"""OT config 5 (20k x 20k, eps 0.01) loop breakdown: per-phase n_i, scan vs host time."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

inst = otprg.gen_random_ot_rational(20000, 20000, 1)
for rep in range(3):
    t0 = time.perf_counter()
    plan, st = otprg.solve_ot(inst, 0.01)
    wall = (time.perf_counter() - t0) * 1e3
    d = st.device
    print(f"wall {wall:.1f} build {d['build_ms']:.1f} loop {d['loop_ms']:.1f} scan {d['scan_ms']:.1f} "
          f"solve {d['solve_ms']:.1f} phases {st.phases} launches {d['gpu_launches']} "
          f"free {list(st.free_counts)}", flush=True)
