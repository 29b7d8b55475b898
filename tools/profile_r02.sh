#!/bin/bash
# Round-2 ncu evidence (run on the GPU box via gpurun):
#  1. one-pass counters of every kernel of one 4096-frame C4 step, per launch
#     plan (fused two-launch plan, fused one-launch plan, staged v1 kernels)
#  2. --set full of the two k_detect launches of one chunk (source-level)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum
for v in "fused:" "onelaunch:fuse_pyramid=0" "staged:staged=1" ${EXTRA_PLANS}; do
  name=${v%%:*}; plan=${v#*:}
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M \
    --csv --log-file gpurun_out/cnt_$name.csv python tools/counters.py --plan "$plan" \
    > gpurun_out/cnt_$name.log 2>&1
  echo "== $name ($plan)"; python tools/counters_summary.py gpurun_out/cnt_$name.csv
done
if [ -z "${NO_FULL}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 6 -c 2 \
    -o gpurun_out/prof_full -f python bench.py --global-batch 4096 --steps 1 --warmup 3 --e2e-steps 1 \
    --no-cpu-baseline --no-parity --no-extras > gpurun_out/ncu_full.log 2>&1
  tail -2 gpurun_out/ncu_full.log
fi
