#!/bin/bash
# Occupancy experiment: default build (3 CTAs/SM) vs a 4-CTA register budget.
mkdir -p gpurun_out
SWEEP_R="${SWEEP_R3:-20}" bash tools/sweep.sh
FLKB_NVCC_FLAGS="-DFLKB_MIN_BLOCKS=${MB:-4}" python -m paper_2003_13493_b200.build --force > gpurun_out/build2.log 2>&1
echo "== MIN_BLOCKS=${MB:-4}" | tee -a gpurun_out/sweep.log
SWEEP_R="${SWEEP_R4:-12 14}" bash tools/sweep.sh
python -m paper_2003_13493_b200.build --force > /dev/null 2>&1
