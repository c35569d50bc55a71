"""Pageable-input H2D: packer thread sweep vs pinning the caller's pages in
place (cudaHostRegister); OT config 5 build time (3.2 GB f64)."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg  # noqa: E402

print("cpus", os.cpu_count(), flush=True)
inst = otprg.gen_random_ot_rational(20000, 20000, 1)
for th in ("8", "8", "4", "12", "reg", "reg", "8"):
    os.environ.pop("OTPRG_H2D_REGISTER", None)
    if th == "reg":
        os.environ["OTPRG_H2D_REGISTER"] = "1"
    else:
        os.environ["OTPRG_H2D_THREADS"] = th
    t0 = time.perf_counter()
    plan, st = otprg.solve_ot(inst, 0.01)
    wall = (time.perf_counter() - t0) * 1e3
    print(f"{th}: wall {wall:.1f} ms build {st.device['build_ms']:.1f} loop {st.device['loop_ms']:.1f}",
          flush=True)
