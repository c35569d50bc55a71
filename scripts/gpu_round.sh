#!/bin/bash
# One GPU session: tests, smoke, bench, then the ncu captures (each ncu only
# after the same command exited 0 without ncu).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
if [ "$1" == "ncu" ]; then
  timeout 300 python scripts/profile_solve.py > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python scripts/profile_solve.py > gpurun_out/ncu_launch.log 2>&1
  timeout 300 python scripts/profile_solve.py > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:propose_stream|phase_loop" \
      -s 2 -c 2 -o gpurun_out/prof_loop python scripts/profile_solve.py > gpurun_out/ncu_full.log 2>&1
fi
