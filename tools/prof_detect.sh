#!/bin/bash
# ncu --set full of the k_detect launches of one bench step (level-0 launch +
# levels 1-2 launch in the two-launch plan) -> gpurun_out/prof_full.ncu-rep
mkdir -p gpurun_out
B=${B:-1024}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect \
  -s ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/prof_full -f python bench.py --plan debug_geom=1 --global-batch $B --steps 1 --warmup 3 --no-parity \
  --e2e-steps 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
