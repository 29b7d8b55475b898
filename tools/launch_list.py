#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_list.py gpurun_out/launches.csv "command line" > profiles/rNN_launches.txt

Per-launch times are cold-cache and serialised under ncu: compare SHARES of the
detection step, not absolutes (the bench's CUDA-event times are the numbers).
"""
import csv
import sys
from collections import defaultdict


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki]
            name = name.split("(")[0] if "(" in name else name
            agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    det = {k: v for k, v in agg.items() if "synth" not in k and "at::" not in k}
    tot = sum(sum(v) for v in det.values())
    print(f"# ncu launch list: {cmd}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
          "compare shares)")
    print(" share     n  mean us   kernel   (shares over detection kernels; synth/torch excluded)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = 100 * sum(v) / tot if k in det else float("nan")
        print(f"{share:6.1f} {len(v):5d} {sum(v) / len(v):10.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
