"""Dense-input solves from pageable numpy memory (the reference API's form)."""
import sys, time
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

inst = otprg.gen_uniform_square(10000, 1, dense=True)
sv = otprg.Solver(0)
for rep in range(3):
    t0 = time.perf_counter()
    m, s = sv.solve(inst, otprg.AssignmentOptions(eps=0.01))
    print(f"dense 10k pageable: wall {(time.perf_counter() - t0) * 1e3:.1f} ms build {s.device['build_ms']:.1f} "
          f"solve {s.device['solve_ms']:.2f}", flush=True)
