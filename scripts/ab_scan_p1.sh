# A/B of the shard scans (libotprg_prev.so = the build before the change) + sharded tests + a parity sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/t_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/t_sharded.log
rm -f gpurun_out/otf_ab.log
for rep in 1 2; do
  for lib in libotprg_prev.so libotprg.so; do
    OTPRG_LIB=$lib PYTHONPATH=. timeout 300 python scripts/probe_otf_only.py >> gpurun_out/otf_ab.log 2>&1
  done
done
timeout 300 python scripts/sweep_parity.py 150 19 > gpurun_out/sweep.log 2>&1; echo "rc=$?" >> gpurun_out/sweep.log
