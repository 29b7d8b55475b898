#!/bin/bash
# ncu evidence for the side configurations (GPU box, via gpurun): --set full of
# two k_detect launches of a C3 (1080p x4, FAST-12, 16x16 cells) and a C5 (4K
# x5, FAST-10) device batch step, after the first step's launches.
mkdir -p gpurun_out
for c in C3 C5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 12 -c 2 \
    -o gpurun_out/prof_$c -f python tools/other_probe.py $c > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
done
