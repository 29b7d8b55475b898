#!/bin/bash
# A/B of library builds on the same box: tools/ab_lib.sh gpurun_out/libA.so gpurun_out/libB.so ...
# Each file is copied over paper_2003_13493_b200/libfastlk_b200.so and timed twice, interleaved.
LIB=paper_2003_13493_b200/libfastlk_b200.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do
  for f in "$@"; do
    cp "$f" $LIB
    timeout 300 python bench.py --no-cpu-baseline --no-extras --e2e-steps 1 --steps 60 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value']), 'fps')"
  done
done
cp /tmp/lib_orig.so $LIB
