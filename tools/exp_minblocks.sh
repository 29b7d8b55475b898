#!/bin/bash
# Occupancy experiment: default build (3 CTAs/SM) vs a 2-CTA register budget.
mkdir -p gpurun_out
SWEEP_R="20" bash tools/sweep.sh
FLKB_NVCC_FLAGS="-DFLKB_MIN_BLOCKS=2" python -m paper_2003_13493_b200.build --force > gpurun_out/build2.log 2>&1
echo "== MIN_BLOCKS=2" | tee -a gpurun_out/sweep.log
SWEEP_R="20 24 32" bash tools/sweep.sh
python -m paper_2003_13493_b200.build --force > /dev/null 2>&1
