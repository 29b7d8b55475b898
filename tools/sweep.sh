#!/bin/bash
# Band-height sweep of the fused kernel (FLKB_BAND_ROWS), short bench runs.
mkdir -p gpurun_out
for R in ${SWEEP_R:-16 20 24 32}; do
  FLKB_BAND_ROWS=$R timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-extras \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R=$R', round(d['value']), 'fps', round(d['roofline']['frac']*100,2), '% roofline', d['ms_per_step'], 'ms/step')"
done 2>&1 | tee gpurun_out/sweep.log
