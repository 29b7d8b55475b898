#!/bin/bash
# Shape sweep of the fused kernel: SWEEP="R:T ..." forces the launch plan's
# band_rows=R and tiles=T ("auto" = the engine's own choice); short bench runs.
mkdir -p gpurun_out
for S in ${SWEEP:-auto 16:1 20:1 24:1 32:1}; do
  if [ "$S" = auto ]; then PL="debug_geom=1"; else PL="band_rows=${S%:*},tiles=${S#*:},debug_geom=1"; fi
  timeout 300 python bench.py --plan "$PL" --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-parity --no-extras 2>gpurun_out/sweep_err.log \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$S', round(d['value']), 'fps', round(d['roofline']['frac']*100,2), '% roofline', d['ms_per_step'], 'ms/step')"
  sort -u gpurun_out/sweep_err.log | grep flkb | tail -3
done 2>&1 | tee -a gpurun_out/sweep.log
