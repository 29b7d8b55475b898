#!/bin/bash
# ncu evidence for profiles/: launch list of a bench run (cold, serialized per-launch
# times: compare shares, not absolutes) and one --set full capture of k_detect.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --batch 4096 --steps 2 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 3 -c 1 \
  -o gpurun_out/prof_full python bench.py --batch 4096 --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_pyramid_down -s 2 -c 1 \
  -o gpurun_out/prof_pyr python bench.py --batch 4096 --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/ncu_pyr.log 2>&1
