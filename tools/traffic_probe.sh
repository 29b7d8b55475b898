#!/bin/bash
# DRAM bytes of the k_detect launches of one C4 step per pyramid_chunk plan value
mkdir -p gpurun_out
for c in ${CHUNKS:-0 4096 512}; do
  if [ "$c" = 0 ]; then n=30; else n=$(( 2 * (4096 + c - 1) / c )); fi
  PYR_CHUNK=$c timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --cache-control none --clock-control none -k regex:k_detect -s $n -c $n --csv \
    --log-file gpurun_out/traffic_$c.csv python tools/traffic_probe.py > gpurun_out/traffic_$c.log 2>&1
  python - $c <<'PY'
import csv, sys
c = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/traffic_{c}.csv")) if r]
h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hd = rows[h]; mi, vi, ui = hd.index("Metric Name"), hd.index("Metric Value"), hd.index("Metric Unit")
tot = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for r in rows[h + 1:]:
    tot[r[mi]] = tot.get(r[mi], 0) + float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
print(c, {k: round(v / 4096) for k, v in tot.items()}, "bytes per frame")
PY
done
