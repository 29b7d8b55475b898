"""The bench's side lines (C2 latency, C1, C3, C5) alone: python tools/other_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

out = bench.other_configs(0)
for k, v in out.items():
    print(k, json.dumps({kk: round(vv, 1) for kk, vv in v.items() if isinstance(vv, (int, float))}))
