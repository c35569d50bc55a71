#!/bin/bash
# Measurement session after the static-slot phase loop (round 2, third part):
# GPU suite, smoke, bench line, configs, per-phase timeline, then ncu (launch
# list of the config-2 solve and one --set full capture of the phase loop;
# each ncu command ran clean without ncu first, in this call).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo "rc=$?" >> gpurun_out/configs.err
for s in 1 2 3; do timeout 120 python scripts/timeline.py 10000 0.01 $s u16; done > gpurun_out/timeline.txt 2>&1
if [ "$1" == "ncu" ]; then
  python scripts/profile_solve.py > gpurun_out/plain.log 2>&1 &&
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_solve.csv \
      python scripts/profile_solve.py > gpurun_out/ncu_launch.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:phase_loop -s 2 -c 2 \
      -o gpurun_out/prof_loop python scripts/profile_solve.py > gpurun_out/ncu_loop.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_loop.log
fi
