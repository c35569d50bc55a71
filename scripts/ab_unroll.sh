# A/B of the shared-t scan unroll (OTPRG_UNROLL_SMEM: 128-bit loads in flight per lane)
for rep in 1 2; do
  PYTHONPATH=. python scripts/ab_lib.py
  for u in 2 4 6; do OTPRG_LIB=libotprg_c16_l2_u${u}_b512.so PYTHONPATH=. python scripts/ab_lib.py; done
done
