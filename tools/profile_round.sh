#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box via gpurun):
#  1. launch list of a default-shaped bench run (cold, serialised per-launch
#     times: compare shares, not absolutes)
#  2. --set full of the two k_detect launches of one 4096-frame step
#     (level-0 launch with the fused pyramid, then levels 1-2)
#  3. --set full of the session kernels (k_track, k_template) on the bench's
#     session sequence
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --global-batch 4096 --no-parity --steps 2 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 6 -c 2 \
  -o gpurun_out/prof_full -f python bench.py --global-batch 4096 --no-parity --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline --no-extras > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_track|k_template" \
  -s 20 -c 4 -o gpurun_out/prof_lk -f python -c "
import bench, paper_2003_13493_b200 as fl
frames = bench.session_frames(0)
s = fl.Session(fl.Config(**bench.SESSION_CFG))
for f in frames[:30]:
    s.process(f)
" > gpurun_out/ncu_lk.log 2>&1
for f in gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/ncu_lk.log; do tail -n 2 $f; done
