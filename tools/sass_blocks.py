#!/usr/bin/env python
"""SASS basic blocks (runs of instructions with the same execution count) of
each captured k_detect launch by executed warp instructions, and the share of
instructions and stall samples in code executed once per warp (per-CTA setup,
scans, barriers, flush) vs the loops (ncu source page, SASS view).

    python tools/sass_blocks.py gpurun_out/prof_full.ncu-rep [launches] [top]
"""
import csv
import io
import subprocess
import sys


def launch(rep, i):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(i), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
    ism = hdr.index("Warp Stall Sampling (All Samples)")
    ins, seen = [], set()
    for r in rows[rows.index(hdr) + 1:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        if a in seen:  # the page repeats the listing
            break
        seen.add(a)
        ins.append((a, r[isrc].strip(), int(r[iex]), int(r[ism])))
    return ins


def main(rep, launches=2, top=16):
    for li in range(int(launches)):
        ins = launch(rep, li)
        base, warps = ins[0][0], ins[0][2]
        tot = sum(e for _, _, e, _ in ins) or 1
        tots = sum(s for *_, s in ins) or 1
        groups = []
        for a, s, e, sm in ins:
            if groups and groups[-1][2] == e:
                g = groups[-1]
                g[1], g[3], g[4] = a, g[3] + 1, g[4] + sm
            else:
                groups.append([a, a, e, 1, sm, s])
        print(f"== launch {li}: {len(ins)} SASS instructions, {tot} warp-instr executed, "
              f"{tot / warps:.0f} per warp ({warps} warps)")
        cls = {}
        for a, s, e, sm in ins:
            r = e / warps
            k = "once per warp" if 0.9 <= r <= 1.01 else ("< once" if r < 0.9 else "loops")
            c = cls.setdefault(k, [0, 0])
            c[0] += e
            c[1] += sm
        for k, (e, sm) in cls.items():
            print(f"  {k:14s} {100 * e / tot:5.1f}% inst {100 * sm / tots:5.1f}% stall samples")
        for g in sorted(groups, key=lambda g: -g[2] * g[3])[:int(top)]:
            print(f"  {100 * g[2] * g[3] / tot:5.2f}% inst {100 * g[4] / tots:5.2f}% smp  "
                  f"{g[0] - base:#07x}-{g[1] - base:#07x} len {g[3]:4d} x{g[2] / warps:5.2f}/warp  {g[5][:48]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
