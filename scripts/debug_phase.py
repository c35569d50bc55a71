"""Phase-by-phase GPU vs oracle comparison for one square instance."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

n, eps, seed = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
o = Oracle.get()
cost = o.gen_uniform_square(n, seed)
k, uf, uc = o.scale_round_costs(cost, eps)
inst = otprg.gen_uniform_square(n, seed)
sc = otprg.scale_round_costs(inst, eps)
print("k mismatches:", int((sc.k != k).sum()), flush=True)
kT = k.T.copy()
# oracle phase-by-phase
ya = np.zeros(n, np.int64); yb = np.ones(n, np.int64); ma = -np.ones(n, np.int64); mb = -np.ones(n, np.int64)
S = otprg.Solver(0)
S.prepare(inst, eps)
S.begin()
for p in range(1, 40):
    bfree = np.nonzero(mb == -1)[0]
    if len(bfree) <= np.floor(eps * n):
        break
    claimed = set(); prime = []
    for b in bfree:
        adm = np.nonzero(ya + yb[b] == kT[b] + 1)[0]
        for a in adm:
            if a not in claimed:
                claimed.add(a); prime.append((a, b)); break
    pb = set()
    for a, b in prime:
        if ma[a] != -1: mb[ma[a]] = -1
        ma[a] = b; mb[b] = a; ya[a] -= 1; pb.add(b)
    for b in bfree:
        if b not in pb: yb[b] += 1
    done, fin = S.step(p)
    m, s = S.snapshot()
    bad_a = np.nonzero(m.match_of_a != ma)[0]
    print(f"phase {p}: n_i={len(bfree)} |M'|={len(prime)} gpu_free_next={s.free_counts[-1] if len(s.free_counts) else None} "
          f"match_mismatch={len(bad_a)} ya_mis={(s.duals_final.y_a != ya).sum()} yb_mis={(s.duals_final.y_b != yb).sum()}", flush=True)
    if len(bad_a):
        for a in bad_a[:5]:
            print("   a", a, "gpu b", m.match_of_a[a], "oracle b", ma[a])
        gb = set(np.nonzero(m.match_of_b != mb)[0][:10])
        for b in list(gb)[:5]:
            adm = np.nonzero(kT[b] == 0)[0] if p == 1 else None
            print("   b", b, "gpu a", m.match_of_b[b], "oracle a", mb[b], "adm", adm[:10] if adm is not None else None)
        break
