"""The bench's batch side lines (C1, C3, C5) alone, device-resident, no CPU
baselines: python tools/other_probe.py [name ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

names = sys.argv[1:] or ["C1", "C3", "C5"]
for name in names:
    r = bench.side_config(name, bench.SIDE_CONFIGS[name], 0, bench.hbm_peak()[0], cpu=False)
    print(name, round(r["frames_per_s"]), "frames/s", "kernel_us", round(r["roofline"]["kernel_us_per_step"], 1))
