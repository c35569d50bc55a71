"""Per-step timeline of the persistent OT phase loop (OTPRG_OT_STEPTIME=1):
block 0's time per barrier-delimited step, summed over the solve (stderr)."""
import os
import sys
sys.path.insert(0, ".")
os.environ["OTPRG_OT_STEPTIME"] = "1"
import paper_2203_03732_b200 as otprg  # noqa: E402

for n in (int(x) for x in (sys.argv[1:] or ["100", "1000"])):
    inst = otprg.gen_random_ot_rational(n, n, 1)
    for _ in range(2):
        plan, st = otprg.solve_ot(inst, 0.01)
    print(f"n={n}: phases {st.phases} loop {st.device['loop_ms']:.2f} ms", flush=True)
