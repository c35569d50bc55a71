"""Lockstep u16 vs u32 solves: first phase where the states differ."""
import numpy as np
import paper_2203_03732_b200 as otprg

for n, seed, eps in ((64, 1, 0.05),):
    inst = otprg.gen_uniform_square(n, seed)
    svs = {}
    for st in ("u16", "u32"):
        sv = otprg.Solver(0)
        sv.prepare(inst, eps, st)
        sv.begin()
        svs[st] = sv
    k = otprg.Solver(0).scale_round_costs(inst, eps, "u16").k
    phase = 0
    while phase < 10:
        snaps = {}
        for st, sv in svs.items():
            done, fin = sv.step(phase + 1)
            snaps[st] = sv.snapshot()
        phase += 1
        (m1, s1), (m2, s2) = snaps["u16"], snaps["u32"]
        da = np.nonzero(s1.duals_final.y_a != s2.duals_final.y_a)[0]
        db = np.nonzero(s1.duals_final.y_b != s2.duals_final.y_b)[0]
        dm = np.nonzero(m1.match_of_a != m2.match_of_a)[0]
        print("phase", phase, "diff y_a", da[:8], "y_b", db[:8], "match_a", dm[:8])
        if len(da) or len(db) or len(dm):
            for b in db[:4]:
                print(" b", b, "yb16", s1.duals_final.y_b[b], "yb32", s2.duals_final.y_b[b],
                      "row k+ya(u16) min", int((k[:, b] + s1.duals_final.y_a).min()),
                      "adm16", np.nonzero(k[:, b] + 1 == s1.duals_final.y_a + s1.duals_final.y_b[b] - 0)[0][:5])
            for a in da[:4]:
                print(" a", a, "ya16", s1.duals_final.y_a[a], "ya32", s2.duals_final.y_a[a],
                      "m16", m1.match_of_a[a], "m32", m2.match_of_a[a])
            for a in dm[:4]:
                print(" m a", a, "m16", m1.match_of_a[a], "m32", m2.match_of_a[a])
            break
    sc32 = otprg.Solver(0).scale_round_costs(inst, eps, "u32").k
    print("k equal", np.array_equal(k, sc32))
