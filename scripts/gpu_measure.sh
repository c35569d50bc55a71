#!/bin/bash
# One measurement session (round 2, second half): the GPU suite, smoke, the
# bench line, the other configs, then ncu (each ncu after the same command
# ran clean without it).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo "rc=$?" >> gpurun_out/configs.err
timeout 600 python scripts/ot_small_ab.py > gpurun_out/ot_small_ab.log 2>&1
if [ "$1" == "ncu" ]; then
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:l1_round -c 1 -o gpurun_out/ncu_l1_round \
      python scripts/l1_once.py 10000 1 > gpurun_out/ncu_l1.log 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:round_points -c 2 -o gpurun_out/ncu_k2 \
      python scripts/k2_once.py 100000 u16 > gpurun_out/ncu_k2.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_ot.csv \
      python scripts/ot_once.py 20000 > gpurun_out/ncu_ot.log 2>&1
fi
