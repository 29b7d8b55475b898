#!/bin/bash
# Session-line A/B of library builds: tools/session_ab_lib.sh ab_libs/a.so ab_libs/b.so
LIB=paper_2003_13493_b200/libfastlk_b200.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do
  for f in "$@"; do
    cp "$f" $LIB
    python -c "
import bench
d = bench.session_line(0)
o = bench.other_configs(0)
print('$f', round(d['us_per_frame_median'], 1), 'us/frame', {k: round(v) for k, v in d['concurrent_sessions_frames_per_s'].items()}, 'C2', round(o['C2_latency']['e2e_us_median'], 1))
"
  done
done
cp /tmp/lib_orig.so $LIB
