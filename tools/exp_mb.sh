#!/bin/bash
# Occupancy experiment on the GPU box: rebuild with each FLKB_MIN_BLOCKS in $MBS
# (register budget + shared-memory target for that many CTAs/SM) and time the
# engine's own shape choice; restores the default build at the end.
mkdir -p gpurun_out
for mb in ${MBS:-6 7 8}; do
  FLKB_NVCC_FLAGS="-DFLKB_MIN_BLOCKS=$mb" python -m paper_2003_13493_b200.build --force > gpurun_out/build_mb.log 2>&1 || { echo "build $mb failed"; tail gpurun_out/build_mb.log; continue; }
  timeout 300 python bench.py --plan debug_geom=1 --no-parity --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-extras 2>gpurun_out/mb_err.log \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MIN_BLOCKS=$mb', round(d['value']), 'fps', d['ms_per_step'], 'ms/step')"
  sort -u gpurun_out/mb_err.log | grep flkb | tail -2
done
python -m paper_2003_13493_b200.build --force > /dev/null 2>&1
