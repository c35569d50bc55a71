# A/B of low-set cache variants (lib/libotprg_c*_l*_u8_b512.so) against libotprg.so, config 2 seeds 1-3
for rep in 1 2; do
  PYTHONPATH=. python scripts/ab_lib.py
  for v in paper_2203_03732_b200/lib/libotprg_c*_b512.so; do
    OTPRG_LIB=$(basename $v) PYTHONPATH=. python scripts/ab_lib.py
  done
done
