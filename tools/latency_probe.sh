#!/bin/bash
# Session per-frame latency (F12) and C2 single-frame latency, from bench.py's helpers.
python - <<'PY'
import bench
d = bench.session_line(0)
print('session', round(d['us_per_frame_median'], 1), 'us/frame', d['stage_us_median'], 'cold', round(d['cold_start_us']))
o = bench.other_configs(0)
print('C2', round(o['C2_latency']['e2e_us_median'], 1), 'us median,', round(o['C2_latency']['e2e_us_p95'], 1), 'p95')
PY
