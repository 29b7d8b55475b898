#!/bin/bash
# compute-sanitizer over tools/sanitize.py, one tool at a time -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  SANITIZE_TOOL=$tool timeout 1200 compute-sanitizer --tool $tool --print-limit 400 --error-exitcode 9 python tools/sanitize.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize driver ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
