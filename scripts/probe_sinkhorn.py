"""Sinkhorn baseline: device vs the reference CPU (oracle/_ref) timing."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402

for n, eps, ref_too in ((2000, 0.05, True), (10000, 0.05, False), (10000, 0.01, False)):
    r = otprg.gen_random_ot_rational(n, n, 1)
    inst = otprg.OTInstance(r.mu, r.nu, r.cost)
    cfg = otprg.SinkhornConfig(reg=otprg.reg_for_eps(eps, n), max_iters=10000)
    otprg.sinkhorn(inst, otprg.SinkhornConfig(reg=0.1, max_iters=2), entries=False)  # warm
    t0 = time.perf_counter()
    res = otprg.sinkhorn(inst, cfg, entries=False)
    wall = (time.perf_counter() - t0) * 1e3
    d = res.device
    line = (f"n={n} eps={eps} reg={cfg.reg:.3g}: gpu {wall:.1f} ms (build {d['build_ms']:.1f}, loop "
            f"{d['loop_ms']:.1f}, round {d['round_ms']:.1f}) iters {res.iters} conv {res.converged} "
            f"cost {res.cost:.12g} per-iter {d['loop_ms'] / max(res.iters, 1):.3f} ms")
    if ref_too:
        L = Reference.get().lib
        L.ref_sinkhorn.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                   C.c_int32, C.c_double] + [C.c_void_p] * 8 + [C.c_int64, C.c_void_p]
        it, cv, vi, pc, ms, ne = C.c_int32(), C.c_int32(), C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        cost = np.ascontiguousarray(r.cost)
        st = L.ref_sinkhorn(n, n, r.mu.ctypes.data, r.nu.ctypes.data, cost.ctypes.data, cfg.reg, 10000, 1e-9,
                            C.byref(it), C.byref(cv), C.byref(vi), C.byref(pc), C.byref(ne), None, None, None, 0,
                            C.byref(ms))
        line += f" | reference {ms.value:.1f} ms iters {it.value} cost {pc.value:.12g} (st {st})"
    print(line, flush=True)
