#!/bin/bash
# A/B timing of launch-plan variants: tools/ab.sh "fuse_pyramid=0" "fuse_pyramid=1" ...
# (each argument is passed as bench.py --plan; "" = the automatic plan)
# Each variant's bench line -> gpurun_out/ab_<i>.json; a summary on stdout.
mkdir -p gpurun_out
i=0
for v in "$@"; do
  timeout 300 python bench.py --plan "$v" --no-cpu-baseline --no-parity --no-extras --e2e-steps 2 ${BENCH_ARGS} \
    > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$v" gpurun_out/ab_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{sys.argv[1]:40s} fps={d['value']:.0f} detect_us={r['kernel_us_per_step']:.1f} "
          f"other={r['other_kernels_us']} e2e={d['e2e']['value']:.0f} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  i=$((i+1))
done
