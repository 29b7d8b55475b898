#!/usr/bin/env python
"""Executed-instruction and stall-sample shares per phase of the fused kernel,
per captured launch (ncu source page; `// --- N.` markers in kernels_fused.cuh
delimit the phases; helpers above the kernel are attributed by name).

    python tools/phase_split.py gpurun_out/prof_full.ncu-rep [launches]
"""
import csv
import io
import re
import subprocess
import sys

SRC = "paper_2003_13493_b200/csrc/kernels_fused.cuh"
HELPERS = {"transpose32x8": "2. planes", "sliced_less": "3. masks", "sliced_arc": "3. masks",
           "and3": "3. masks", "or3": "3. masks", "lop3_": "3. masks", "shr_fma": "2-3 shifts",
           "shl_fma": "2-3 shifts", "shift_fma": "2-3 shifts", "sad_b_packed": "4c. score",
           "vabsdiff4_acc": "4c. score", "FastDiv": "div", "TaskIter": "2-3 task walk"}
SUB4 = [("4a. count+scan", "const int tasks_f"), ("4b. list build", "auto build = [&](int w0)"),
        ("4c. score", "const uint32_t rp_magic = RADIUS"), ]
SUB5 = [("5a. nms", "// --- 5."), ("5b. cell keys", "if (!keep) continue;")]


def phase_map():
    lines = open(SRC).read().split("\n")
    kstart = next(i for i, l in enumerate(lines) if l.startswith("template <int N, int KIND, int RADIUS, bool STATS>"))
    ph, cur, func = {}, "0. setup", None
    for i, l in enumerate(lines):
        m = re.search(r"// --- (\d\w?)\.\s*(\w+)", l)
        if m and i > kstart:
            cur = f"{m.group(1)}. {m.group(2)}"
        for name, marker in SUB4 + SUB5:
            if marker in l and i > kstart:
                cur = name
        if i < kstart:
            for h, p in HELPERS.items():
                if re.search(r"\b" + h, l) and ("__device__" in l or "struct" in l):
                    func = p
            ph[i + 1] = func or "helpers"
        else:
            ph[i + 1] = cur
    return ph


def source(rep, launch):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "--launch-skip", str(launch), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    agg, cur, hdr = {}, None, None
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            agg[(cur, int(r[0]))] = (int(r[7]), int(r[6]))
        except ValueError:
            pass
    return agg


def main(rep, launches=2):
    ph = phase_map()
    for li in range(int(launches)):
        agg = source(rep, li)
        ti = sum(v[0] for v in agg.values()) or 1
        ts = sum(v[1] for v in agg.values()) or 1
        out = {}
        for (f, ln), v in agg.items():
            key = ph.get(ln, "other") if f == SRC.split("/")[-1] else f"({f})"
            a = out.setdefault(key, [0, 0])
            a[0] += v[0]
            a[1] += v[1]
        print(f"== launch {li}: share of executed warp instructions / of stall samples")
        for k, v in sorted(out.items(), key=lambda kv: -kv[1][0]):
            if v[0] / ti > 0.002 or v[1] / ts > 0.002:
                print(f"  {k:24s} {100 * v[0] / ti:5.1f}% inst  {100 * v[1] / ts:5.1f}% samples")


if __name__ == "__main__":
    main(*sys.argv[1:])
