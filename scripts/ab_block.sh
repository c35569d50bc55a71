# A/B of the phase-loop block size (OTPRG_BLOCK) at the default unroll
for rep in 1 2; do
  PYTHONPATH=. python scripts/ab_lib.py
  for b in 256 1024; do OTPRG_LIB=libotprg_c16_l2_u4_b${b}.so PYTHONPATH=. python scripts/ab_lib.py; done
done
