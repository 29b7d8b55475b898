#!/bin/bash
# Shape sweep of the fused kernel: SWEEP="R:T ..." forces FLKB_BAND_ROWS=R and
# FLKB_TILES=T ("auto" = the engine's own choice); short bench runs.
mkdir -p gpurun_out
for S in ${SWEEP:-auto 16:1 20:1 24:1 32:1}; do
  if [ "$S" = auto ]; then ENVS=""; else ENVS="FLKB_BAND_ROWS=${S%:*} FLKB_TILES=${S#*:}"; fi
  env $ENVS FLKB_DEBUG_GEOM=1 timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-extras 2>gpurun_out/sweep_err.log \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$S', round(d['value']), 'fps', round(d['roofline']['frac']*100,2), '% roofline', d['ms_per_step'], 'ms/step')"
  sort -u gpurun_out/sweep_err.log | grep flkb | tail -3
done 2>&1 | tee -a gpurun_out/sweep.log
