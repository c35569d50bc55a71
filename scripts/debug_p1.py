"""Phase-1 determinism probe: repeat phase 1, diff against the serial greedy."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

n, eps, seed, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
o = Oracle.get()
k, uf, uc = o.scale_round_costs(o.gen_uniform_square(n, seed), eps)
kT = k.T.copy()
adm = [np.nonzero(kT[b] == 0)[0] for b in range(n)]
claimed = {}
sd = -np.ones(n, np.int64)
for b in range(n):
    for a in adm[b]:
        if a not in claimed:
            claimed[a] = b; sd[b] = a; break
S = otprg.Solver(0)
inst = otprg.gen_uniform_square(n, seed)
S.prepare(inst, eps)
for r in range(reps):
    S.begin()
    S.step(1)
    m, s = S.snapshot()
    gb = m.match_of_b.astype(np.int64)
    diff = np.nonzero(gb != sd)[0]
    print(f"rep {r}: |M'| gpu={int((gb>=0).sum())} sd={int((sd>=0).sum())} diff_b={len(diff)}", flush=True)
    for b in diff[:6]:
        print(f"   b={b} gpu_a={gb[b]} sd_a={sd[b]} adm={list(adm[b][:8])} "
              f"gpu_holder_of_sd_a={m.match_of_a[sd[b]] if sd[b]>=0 else None}", flush=True)
