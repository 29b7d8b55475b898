#!/bin/bash
# One GPU round: parity tests, smoke, bench, ncu launch list (+ optional full capture).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpuinfo.txt 2>&1
nproc >> gpurun_out/gpuinfo.txt
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --batch 512 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
if [ -n "${NCU_FULL}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_detect -s 3 -c 1 -o gpurun_out/prof_full python bench.py --batch 512 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_full.log 2>&1
fi
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log; do echo "== $f"; tail -n 4 $f; done
