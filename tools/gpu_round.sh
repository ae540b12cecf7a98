#!/bin/bash
# One GPU session: tests, smoke, bench lines, ncu launch list + one full capture.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [tests|notests]
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.txt
fi
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --workload mlp784 --steps 50 > gpurun_out/${TAG}_bench_mlp784.json 2>&1; echo "bench784 rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench_mlp784.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch_stdout.txt 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 12 -c 3 -o gpurun_out/${TAG}_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full_stdout.txt 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out | tail -20
