# A/B of the slab scan's loads in flight per lane (OTPRG_SHARD_UNROLL), config 4 sharded G=1
for rep in 1 2; do
  for lib in libotprg.so libotprg_su12.so libotprg_su16.so libotprg_su24.so; do
    OTPRG_LIB=$lib PYTHONPATH=. python scripts/probe_shard_overhead.py 2>&1 | tail -1 | sed "s/^/$lib: /"
  done
done
