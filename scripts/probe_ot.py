"""Config-5 timing probe: GPU solve_ot vs the reference CPU on the same instance."""
import sys
import time
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

for n, eps in ((1000, 0.01), (5000, 0.01), (20000, 0.01)):
    inst = otprg.gen_random_ot_rational(n, n, 1)
    for rep in range(2):
        t0 = time.perf_counter()
        plan, st = otprg.solve_ot(inst, eps)
        wall = (time.perf_counter() - t0) * 1e3
    d = st.device
    print(f"n={n} eps={eps}: phases={st.phases} entries={len(plan.a)} wall={wall:.1f}ms "
          f"build={d['build_ms']:.1f} loop={d['loop_ms']:.1f} scan={d['scan_ms']:.1f} "
          f"launches={d['gpu_launches']} cost={plan.cost!r}", flush=True)
