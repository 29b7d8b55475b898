#!/bin/bash
# CTA-shape experiment: VARIANTS="threads:minblocks:shapes ..." where shapes is
# a comma list of R:T (or auto) handed to tools/sweep.sh.
mkdir -p gpurun_out; : > gpurun_out/sweep.log
for V in ${VARIANTS:-256:3:auto 128:6:auto}; do
  IFS=: read -r TH MB SH <<< "$V"
  FLKB_NVCC_FLAGS="-DFLKB_THREADS=$TH -DFLKB_MIN_BLOCKS=$MB" python -m paper_2003_13493_b200.build --force > gpurun_out/build2.log 2>&1
  echo "== ${TH}x${MB}" >> gpurun_out/sweep.log
  SWEEP="${SH//,/ }" bash tools/sweep.sh
done
python -m paper_2003_13493_b200.build --force > /dev/null 2>&1
