"""OT on the assignment-as-OT form (uniform masses): phase costs."""
import sys, time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

for n, eps in ((1000, 0.05), (1000, 0.1), (2000, 0.05)):
    inst = otprg.gen_uniform_square(n, 1, dense=True)
    ot = otprg.OTInstance(np.full(n, 1.0 / n), np.full(n, 1.0 / n), inst.cost)
    t0 = time.perf_counter()
    plan, st = otprg.solve_ot(ot, eps)
    wall = (time.perf_counter() - t0) * 1e3
    d = st.device
    print(f"n={n} eps={eps}: wall {wall:.1f} ms phases {st.phases} loop {d['loop_ms']:.1f} scan {d['scan_ms']:.1f} "
          f"build {d['build_ms']:.1f} launches {d.get('gpu_launches')} cost {plan.cost}", flush=True)
