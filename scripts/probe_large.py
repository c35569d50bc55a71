"""Large-n assignment probe (config 4 on one GPU): build + solve times, invariants."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

S = otprg.Solver(0)
for n in [int(x) for x in sys.argv[1:]] or [20000, 50000, 100000]:
    inst = otprg.gen_uniform_square(n, 1)
    t0 = time.perf_counter()
    info = S.prepare(inst, 0.01)
    t_prep = (time.perf_counter() - t0) * 1e3
    for rep in range(2):
        m, s = S.solve_prepared()
    d = s.device
    m.validate()
    ok = (m.match_of_a >= 0).all()
    print(f"n={n}: prep_wall={t_prep:.1f}ms build={info['build_ms']:.1f}ms phases={s.phases} "
          f"sum_ni={s.sum_ni} solve={d['solve_ms']:.2f}ms phase1={d['phase1_ms']:.3f}ms "
          f"loop={d['loop_ms']:.2f}ms touched={d['bytes_touched']/1e9:.2f}GB alg={d['bytes_alg']/1e9:.2f}GB "
          f"perfect={ok} cost={d['cost']!r} stats={d['chain_stats']}", flush=True)
