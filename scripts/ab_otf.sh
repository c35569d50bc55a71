# A/B of the on-the-fly tile (OTPRG_OTF_ROWS rows per block, OTPRG_OTF_GU groups per warp step)
for rep in 1 2; do
  for lib in libotprg.so libotprg_otf_r8_g4.so libotprg_otf_r32_g4.so libotprg_otf_r16_g8.so libotprg_otf_r16_g2.so; do
    OTPRG_LIB=$lib PYTHONPATH=. python scripts/probe_otf_only.py
  done
done
