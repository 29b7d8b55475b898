#!/bin/bash
# Round-2 closing evidence (GPU box, via gpurun): GPU tests, sanitizers, the
# one-pass counters of a C4 step's k_detect launches (DRAM / L2 bytes and
# instructions per frame), the ncu launch list, --set full of one chunk's two
# k_detect launches, and the default bench line.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; tail -2 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash tools/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; cat gpurun_out/sanitize_summary.txt
CHUNKS=0 bash tools/traffic_probe.sh > gpurun_out/traffic_summary.txt 2>&1; tail -1 gpurun_out/traffic_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --global-batch 4096 --steps 2 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline --no-parity --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 6 -c 2 \
  -o gpurun_out/prof_full -f python bench.py --global-batch 4096 --steps 1 --warmup 3 --e2e-steps 1 \
  --no-cpu-baseline --no-parity --no-extras > gpurun_out/ncu_full.log 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -c 400 gpurun_out/bench_final.json
