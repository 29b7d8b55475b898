#!/bin/bash
# --set full of the tracking session's kernels (k_track, k_template) on the
# bench's F12 session sequence (GPU box, via gpurun) -> gpurun_out/prof_lk.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_track|k_template" \
  -s 20 -c 4 -o gpurun_out/prof_lk -f python -c "
import bench, paper_2003_13493_b200 as fl
frames = bench.session_frames(0)
s = fl.Session(fl.Config(**bench.SESSION_CFG))
for f in frames[:30]:
    s.process(f)
" > gpurun_out/ncu_lk.log 2>&1
tail -n 2 gpurun_out/ncu_lk.log
