# A/B of the persistent OT loop's threads per block (OTPRG_OT_THREADS), best of 4 solves
for t in 1024 512 256; do
  OTPRG_OT_THREADS=$t python - <<'PY'
import os, sys
sys.path.insert(0, ".")
import paper_2203_03732_b200 as otprg
for n in (100, 1000, 5000, 20000):
    inst = otprg.gen_random_ot_rational(n, n, 1)
    best = min(otprg.solve_ot(inst, 0.01)[1].device["loop_ms"] for _ in range(4))
    print(f"threads {os.environ['OTPRG_OT_THREADS']} n={n}: loop {best:.2f} ms", flush=True)
PY
done
