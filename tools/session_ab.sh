#!/bin/bash
# A/B of the session line: python bench.py's F12_session under env variants.
for v in "$@"; do
  env $v python -c "
import json, bench
d = bench.session_line(0)
print('$v', round(d['us_per_frame_median'],1), 'us/frame', d['stage_us_median'], 'cold', round(d['cold_start_us']))
"
done
