"""Config 4 sharded (G=1): host time per protocol call vs the device timer, to
split the per-round cost into GPU work and host/launch overhead."""
import collections, sys, time
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2203_03732_b200 as otprg  # noqa: E402
from paper_2203_03732_b200 import sharded as SH  # noqa: E402

acc = collections.defaultdict(float)
cnt = collections.Counter()
for name in ("begin", "top", "scan", "da"):
    orig = getattr(SH.DeviceRank, name)

    def wrap(self, *a, _o=orig, _n=name, **k):
        t0 = time.perf_counter()
        r = _o(self, *a, **k)
        acc[_n] += time.perf_counter() - t0
        cnt[_n] += 1
        return r
    setattr(SH.DeviceRank, name, wrap)

inst = otprg.gen_uniform_square(100_000, 1)
sv = SH.ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01), 1)
for rep in range(4):
    acc.clear(); cnt.clear()
    torch.cuda.synchronize()
    sv.timer_start()
    t0 = time.perf_counter()
    m, s = sv.solve()
    wall = (time.perf_counter() - t0) * 1e3
    dev = sv.timer_stop()
    print(f"rep {rep}: wall {wall:.2f} ms device-timer {dev:.2f} ms phases {s.phases} refills "
          f"{s.device['refill_rounds']} | " + " ".join(f"{k} {acc[k]*1e3:.2f}ms/{cnt[k]}" for k in acc), flush=True)
