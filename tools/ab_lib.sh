#!/bin/bash
# A/B of library builds on the same box: tools/ab_lib.sh ab_libs/libA.so ab_libs/libB.so ...
# Each file is copied over paper_2003_13493_b200/libfastlk_b200.so and timed
# (REPS times, interleaved); every run also checks all 4096 frames against the
# reference build (parity mismatches printed beside the rate).
LIB=paper_2003_13493_b200/libfastlk_b200.so
cp $LIB /tmp/lib_orig.so
for rep in $(seq ${REPS:-3}); do
  for f in "$@"; do
    cp "$f" $LIB
    timeout 300 python bench.py --no-cpu-baseline --no-extras --e2e-steps 1 --steps ${STEPS:-60} ${BENCH_ARGS} 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value']), 'fps', 'kernel_us', round(d['roofline']['kernel_us_per_step'],1), 'mismatches', d.get('parity',{}).get('mismatches'))"
  done
done
cp /tmp/lib_orig.so $LIB
