"""Per-phase device timeline of config-2 solves (tracing on)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
S = otprg.Solver(0)
S.prepare(otprg.gen_uniform_square(n, seed), eps)
S.set_trace(20000)
for _ in range(3):
    m, s = S.solve_prepared()
tr = S.get_trace(s.phases).astype(np.int64)
t0 = tr[:, 0]
start = t0
staged = tr[:, 1] - t0
p_last = tr[:, 2] - t0
p_first = (~tr[:, 3].astype(np.uint64)).astype(np.int64) - t0
b1 = tr[:, 4] - t0
a_last = tr[:, 5] - t0
b2 = tr[:, 6] - t0
nxt = np.append(t0[1:] - t0[:-1], 0)
print(f"solve_ms={s.device['solve_ms']:.3f} loop_ms={s.device['loop_ms']:.3f} phases={s.phases}")
print("phase  n_i  staged  Pfirst  Plast  bar1  Alast  bar2  next   (us from phase start)")
for i in list(range(0, 8)) + list(range(8, s.phases, max(1, s.phases // 25))):
    print(f"{i+1:5d} {tr[i,7]:5d} {staged[i]/1e3:7.2f} {p_first[i]/1e3:7.2f} {p_last[i]/1e3:6.2f} "
          f"{b1[i]/1e3:6.2f} {a_last[i]/1e3:6.2f} {b2[i]/1e3:6.2f} {nxt[i]/1e3:6.2f}")
sl = slice(1, s.phases - 1)
print("means over phases 2..: staged %.2f Pfirst %.2f Plast %.2f bar1 %.2f Alast %.2f bar2 %.2f next %.2f" % tuple(
    x[sl].mean() / 1e3 for x in (staged, p_first, p_last, b1, a_last, b2, nxt)))
