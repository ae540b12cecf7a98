#!/bin/bash
# One GPU session: tests, smoke, bench lines, ncu launch list + a full capture.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [tests|notests]
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.txt
fi
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.txt
for W in vgg16 wide_mlp mlp784; do
  timeout 600 python bench.py --workload $W > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err; echo "bench $W rc=$?"
  timeout 600 python bench.py --workload $W --impl reference > gpurun_out/${TAG}_ref_${W}.json 2>&1; echo "ref $W rc=$?"
done
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/${TAG}_ops_vgg16.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch_stdout.txt 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|halo_conv" -s 0 -c 6 -o gpurun_out/${TAG}_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full_stdout.txt 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 12 -c 2 -o gpurun_out/${TAG}_gemm_wide python bench.py --workload wide_mlp --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full_wide_stdout.txt 2>&1; echo "ncu full wide rc=$?"
ls gpurun_out | grep ${TAG}
# summaries on the box (the merged gpurun_out/ is capped at 64 MiB): keep the
# VGG capture for source-level reading, drop the wide-MLP one after summarising
python tools/summarize_ncu.py ${TAG} vgg16 > /dev/null 2>&1
python tools/summarize_ncu.py ${TAG} wide_mlp gemm_wide > /dev/null 2>&1
cp profiles/${TAG}_ncu.md profiles/${TAG}_gemm_wide_ncu.md profiles/gemm_traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/${TAG}_gemm_wide.ncu-rep
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/${TAG}_gemm.ncu-rep
du -sh gpurun_out
# plan-chooser calibration (profiles/calib_<workload>.json) and its predicted scaling
if [ "${CALIB:-1}" = "1" ]; then
  for W in vgg16 wide_mlp; do
    timeout 900 python tools/calibrate.py $W gpurun_out/calib_${W}.json > gpurun_out/${TAG}_calib_${W}.txt 2>&1; echo "calib $W rc=$?"
  done
fi
