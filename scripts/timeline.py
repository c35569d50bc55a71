"""Per-phase device timeline of a solve (tracing on).

Slots (solve_kernels.cu): 0 phase start, 2/3 last/first block done with the
proposal step (3 stores ~t), 4 after the phase barrier, 1/5/6 slowest warp's
scan / atomic / total ns, 7 n_i, 8 bulk list build done (large phases),
9 last block done with the bulk build.
"""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
storage = sys.argv[4] if len(sys.argv) > 4 else "auto"
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(n, seed), eps, storage)
S.set_trace(20000)
for _ in range(3):
    S.flush_l2()
    m, s = S.solve_prepared()
tr = S.get_trace(s.phases).astype(np.int64)
t0 = tr[:, 0]
p_last = tr[:, 2] - t0
p_first = (~tr[:, 3].astype(np.uint64)).astype(np.int64) - t0
bar = tr[:, 4] - t0
nxt = np.append(t0[1:] - t0[:-1], 0)
scan, atom, warp = tr[:, 1], tr[:, 5], tr[:, 6]
bulk = np.where(tr[:, 8] > 0, tr[:, 8] - t0, 0)
print(f"solve_ms={s.device['solve_ms']:.3f} phase1_ms={s.device['phase1_ms']:.3f} "
      f"loop_ms={s.device['loop_ms']:.3f} phases={s.phases} width={s.device['width']}")
print("phase   n_i   bulk  Pfirst  Plast   bar   next | slowest warp: total  scan  atomic (us) | max/warp: scans walks props")
rows = list(range(0, min(8, s.phases))) + list(range(8, s.phases, max(1, s.phases // 20)))
for i in rows:
    print(f"{i+1:5d} {tr[i,7]:5d} {bulk[i]/1e3:6.2f} {p_first[i]/1e3:7.2f} {p_last[i]/1e3:6.2f} "
          f"{bar[i]/1e3:6.2f} {nxt[i]/1e3:6.2f} | {warp[i]/1e3:6.2f} {scan[i]/1e3:6.2f} {atom[i]/1e3:6.2f} | "
          f"{tr[i,10]:4d} {tr[i,11]:4d} {tr[i,12]:4d}")
sl = slice(1, s.phases - 1)
print("means over phases 2..: Pfirst %.2f Plast %.2f bar %.2f next %.2f | warp %.2f scan %.2f atomic %.2f" % tuple(
    x[sl].mean() / 1e3 for x in (p_first, p_last, bar, nxt, warp, scan, atom)))
print("means over phases 2..: max scans/warp %.2f walks %.2f props %.2f" % tuple(
    tr[sl, j].mean() for j in (10, 11, 12)))
print("chain stats", s.device["chain_stats"], "bytes_touched", s.device["bytes_touched"] / 1e6, "MB")
