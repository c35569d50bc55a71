"""Multi-process check of the sharded protocol on ONE GPU: two torch.distributed
ranks (gloo exchange; both contexts on cuda:0 via OTPRG_DEVICE=0) each own half
the A rows; results must equal the golden pins / the fused solver.  (The
protocol is host-synced, so no kernel waits on another rank's kernel.)

  OTPRG_DEVICE=0 python -m torch.distributed.run --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29555 scripts/dist_on_one_gpu.py
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2203_03732_b200 as otprg  # noqa: E402
from golden_util import PIN_KEYS, pins_of  # noqa: E402
from paper_2203_03732_b200.sharded import ShardedSolver  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
golden = json.load(open("tests/golden/assign_pins.json"))
ok = True
for key, otf in (("square_n4000_eps0.01_s1", False), ("square_n10000_eps0.01_s2", False),
                 ("square_n10000_eps0.1_s1", False), ("square_n4000_eps0.01_s1", True),
                 ("square_n10000_eps0.01_s2", True)):
    w = golden[key]
    inst = otprg.gen_uniform_square(w["n_a"], w["seed"])
    sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=w["eps"]), distributed=True, K=4, on_the_fly=otf)
    t0 = time.perf_counter()
    m, s = sv.solve()
    ms = (time.perf_counter() - t0) * 1e3
    sv.close()
    got = pins_of(m.match_of_a, s.duals_final.y_a, s.duals_final.y_b, s.free_counts, s.phases, s.sum_ni,
                  s.device["cost"])
    same = all(got[k] == w[k] for k in PIN_KEYS)
    ok &= same
    if rank == 0:
        print(f"{key} otf={otf}: world={world} bit-exact={same} phases={s.phases} refills={s.device['refill_rounds']} "
              f"wall={ms:.1f} ms", flush=True)
# n = 100k: the two-rank result equals the fused single-GPU solver
inst = otprg.gen_uniform_square(100_000, 1)
sv = ShardedSolver(inst, otprg.AssignmentOptions(eps=0.01), distributed=True)
m2, s2 = sv.solve()
sv.close()
if rank == 0:
    m1, s1 = otprg.Solver(0).solve(inst, otprg.AssignmentOptions(eps=0.01))
    same = (np.array_equal(m1.match_of_a, m2.match_of_a) and np.array_equal(s1.duals_final.y_a, s2.duals_final.y_a)
            and np.array_equal(s1.duals_final.y_b, s2.duals_final.y_b) and s1.phases == s2.phases)
    ok &= same
    print(f"n=100k two ranks vs fused: identical={same} phases={s2.phases}", flush=True)
flag = torch.tensor([1 if ok else 0])
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print("DIST OK" if flag.item() == 1 else "DIST FAILED", flush=True)
dist.destroy_process_group()
sys.exit(0 if flag.item() == 1 else 1)
