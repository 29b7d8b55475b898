"""Per-kernel totals per frame from a tools/counters.py ncu CSV.

    python tools/counters_summary.py gpurun_out/cnt_fused.csv [frames] [pixels_per_frame]
"""
import csv
import sys
from collections import OrderedDict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "inst": 1, "": 1}


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hd = rows[h]
    ki, mi, vi, ui = (hd.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = hd.index("ID")
    per = OrderedDict()
    launches = {}
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        per.setdefault(name, {}).setdefault(r[mi], 0.0)
        per[name][r[mi]] += v
        launches.setdefault(name, set()).add(r[idi])
    return per, {k: len(v) for k, v in launches.items()}


def main():
    path = sys.argv[1]
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    px = int(sys.argv[3]) if len(sys.argv) > 3 else 473760
    per, nl = load(path)
    tot = {}
    print(f"{'kernel':34s} {'launches':>8s} {'us':>9s} {'dram B/frame':>13s} {'L2 B/frame':>12s} "
          f"{'warp-inst/px':>12s} {'thread-inst/px':>14s}")
    for k, m in per.items():
        for mk, v in m.items():
            tot[mk] = tot.get(mk, 0.0) + v
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        print(f"{k[:34]:34s} {nl[k]:8d} {m.get('gpu__time_duration.sum', 0):9.1f} "
              f"{dram / frames:13.0f} {m.get('lts__t_bytes.sum', 0) / frames:12.0f} "
              f"{m.get('smsp__inst_executed.sum', 0) / frames / px:12.3f} "
              f"{m.get('smsp__thread_inst_executed.sum', 0) / frames / px:14.2f}")
    dram = tot.get("dram__bytes_read.sum", 0) + tot.get("dram__bytes_write.sum", 0)
    print(f"{'TOTAL':34s} {sum(nl.values()):8d} {tot.get('gpu__time_duration.sum', 0):9.1f} "
          f"{dram / frames:13.0f} {tot.get('lts__t_bytes.sum', 0) / frames:12.0f} "
          f"{tot.get('smsp__inst_executed.sum', 0) / frames / px:12.3f} "
          f"{tot.get('smsp__thread_inst_executed.sum', 0) / frames / px:14.2f}")


if __name__ == "__main__":
    main()
