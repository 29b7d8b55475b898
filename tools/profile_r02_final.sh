#!/bin/bash
# Round-2 evidence for profiles/ (GPU box, via gpurun):
#  1. launch list of a default bench step (4096 frames; cold, serialised: shares only)
#  2. --set full of one chunk's two k_detect launches (source-level)
#  3. compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize.py
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline --no-parity --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 6 -c 2 \
  -o gpurun_out/prof_full -f python bench.py --global-batch 4096 --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline --no-parity --no-extras > gpurun_out/ncu_full.log 2>&1
bash tools/sanitize.sh
