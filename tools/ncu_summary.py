#!/usr/bin/env python
"""Summarise an ncu report (from `ncu --set full --import-source on`) for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep [--pixels-per-launch P] [--top 30]

Prints the headline metrics (duration, issue utilisation, occupancy, DRAM
bytes, instructions per pixel) and the source lines that execute the most
warp instructions, with their share of stall samples.
"""
import argparse
import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def raw_metrics(rep):
    out = ncu(["-i", rep, "--page", "raw", "--csv"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, kernels = rows[0], rows[1], rows[2:]
    return [dict(zip(hdr, r)) for r in kernels], dict(zip(hdr, units))


def source_lines(rep):
    out = ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
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
            agg[(cur, int(r[0]))] = (int(r[7]), int(r[6]), r[1].strip())
        except ValueError:
            pass
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--pixels-per-launch", type=str, default="0",
                    help="pixels of each captured launch, comma-separated (one value = all)")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    kernels, units = raw_metrics(a.report)
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__thread_inst_executed_per_inst_executed.ratio",
            "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg"]
    px = [float(v) for v in a.pixels_per_launch.split(",")]
    for li, k in enumerate(kernels):
        print(f"== launch {li}: {k.get('Kernel Name', '?')[:100]}")
        for m in keys:
            if m in k:
                print(f"  {m:62s} {k[m]:>18s} {units.get(m, '')}")
        npx = px[min(li, len(px) - 1)]
        if npx:
            wi = float(k.get("smsp__inst_executed.sum", "0").replace(",", ""))
            tr = float(k.get("smsp__thread_inst_executed_per_inst_executed.ratio", "0").replace(",", ""))
            print(f"  pixels in the launch           {npx:14.0f}")
            print(f"  warp instructions / pixel      {wi / npx:10.3f}")
            print(f"  thread instructions / pixel    {wi * tr / npx:10.1f}")
    print("\n== pipe utilisation (sm__inst_executed_pipe_*.avg.pct_of_peak_sustained_active) and "
          "stall reasons (warps per issued instruction)")
    for li, k in enumerate(kernels):
        pipes = {m.split("pipe_")[1].split(".")[0]: float(v.replace(",", "")) for m, v in k.items()
                 if m.startswith("sm__inst_executed_pipe_") and m.endswith(".avg.pct_of_peak_sustained_active")
                 and "subpipe" not in m and "type" not in m and v.strip()}
        stalls = {m.split("stalled_")[1].split("_per_issue")[0]: float(v.replace(",", ""))
                  for m, v in k.items()
                  if m.startswith("smsp__average_warps_issue_stalled_") and v.strip()}
        top_p = sorted(((v, n) for n, v in pipes.items() if v >= 1.0), reverse=True)
        top_s = sorted(((v, n) for n, v in stalls.items() if v >= 0.2), reverse=True)
        print(f"  launch {li} pipes: " + ", ".join(f"{n} {v:.1f}%" for v, n in top_p))
        print(f"  launch {li} stalls: " + ", ".join(f"{n} {v:.2f}" for v, n in top_s))
    agg = source_lines(a.report)
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"\n== top source lines by executed warp instructions (total {tot})")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"  {key[0][:20]:20s}:{key[1]:4d} {100 * v[0] / tot:5.1f}% inst "
              f"{100 * v[1] / ts:5.1f}% samples  {v[2][:80]}")


if __name__ == "__main__":
    sys.exit(main())
