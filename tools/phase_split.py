#!/usr/bin/env python
"""Executed-instruction share per phase of the fused kernel (ncu source page).

Phases are delimited by the '// --- N.' markers in kernels_fused.cuh; helper
functions are attributed to the phase that calls them.
"""
import re
import subprocess
import sys

sys.path.insert(0, "tools")
from ncu_summary import source_lines  # noqa: E402

SRC = "paper_2003_13493_b200/csrc/kernels_fused.cuh"
HELPERS = {"transpose32x8": "2 planes", "sliced_less": "3 masks", "sliced_arc": "3 masks",
           "and3": "3 masks", "or3": "3 masks", "lop3_": "3 masks", "sad_b_packed": "4 list+score",
           "vabsdiff4_acc": "4 list+score", "FastDiv": "5 nms+keys", "TaskIter": "2 planes"}


def main(rep):
    lines = open(SRC).read().split("\n")
    phase_of = {}
    cur = "0 setup"
    func = None
    for i, l in enumerate(lines, 1):
        m = re.search(r"// --- (\d)\.\s*(\w+)", l)
        if m:
            cur = f"{m.group(1)} {m.group(2)}"
        for h, ph in HELPERS.items():
            if re.search(r"\b" + h, l) and ("__device__" in l or "struct" in l):
                func = ph
        if l.startswith("template <int N, int KIND, int RADIUS>"):
            func = None
        phase_of[i] = func or cur
    agg = source_lines(rep)
    tot = sum(v[0] for v in agg.values())
    out = {}
    for (f, ln), v in agg.items():
        key = phase_of.get(ln, "other") if f == "kernels_fused.cuh" else f
        out[key] = out.get(key, 0) + v[0]
    for k, v in sorted(out.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / tot:6.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
