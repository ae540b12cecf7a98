#!/bin/bash
# Final round-2 evidence: tests, smoke, bench lines (both arms) for every
# workload, ncu launch list + --set full summaries, elementwise HBM GB/s,
# overlap trace, simulator cross-check, plan-chooser calibration.
set -u
TAG=${TAG:-r02z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
for W in vgg16 resnet18 wide_mlp mlp784 lenet5; do
  timeout 900 python bench.py --workload $W > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err; echo "bench $W rc=$?"
  timeout 900 python bench.py --workload $W --impl reference > gpurun_out/${TAG}_ref_${W}.json 2>&1; echo "ref $W rc=$?"
done
for k in 2 4 8; do
  PPB_BENCH_PLAN_DEVICES=$k timeout 600 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/${TAG}_bench_vgg16_pd$k.json 2>/dev/null; echo "vgg pd$k rc=$?"
done
timeout 600 python bench.py --no-cpu-baseline --steps 50 --m 4 --memory proposed > gpurun_out/${TAG}_bench_vgg16_m4_proposed.json 2>/dev/null; echo "vgg m4 rc=$?"
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/${TAG}_ops_vgg16.jsonl 2>&1
timeout 300 python tools/profile_ops.py resnet18 > gpurun_out/${TAG}_ops_resnet18.jsonl 2>&1
timeout 600 python tools/overlap_trace.py vgg16 4 proposed > gpurun_out/${TAG}_overlap_vgg16_m4.jsonl 2>&1
timeout 600 python tools/sim_crosscheck.py vgg16 --n 1 --Z 1 --m 4 > gpurun_out/${TAG}_simcheck.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|halo_conv" -s 0 -c 6 -o gpurun_out/${TAG}_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 12 -c 2 -o gpurun_out/${TAG}_gemm_wide python bench.py --workload wide_mlp --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu wide rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'pool_fwd|conv_merge|dense_conv|splitk_epilogue|colsum|bias_update|loss_head|im2col|reduce_mask|finalize|residual' --clock-control none --csv --log-file gpurun_out/${TAG}_ew.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/${TAG}_ew.csv > gpurun_out/${TAG}_ew_summary.jsonl
python tools/summarize_ncu.py ${TAG} vgg16 > /dev/null 2>&1
python tools/summarize_ncu.py ${TAG} wide_mlp gemm_wide > /dev/null 2>&1
cp profiles/${TAG}_ncu.md profiles/${TAG}_gemm_wide_ncu.md profiles/gemm_traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/${TAG}_gemm_wide.ncu-rep gpurun_out/${TAG}_gemm.ncu-rep
[ "${CALIB:-1}" = "1" ] && for W in vgg16 wide_mlp; do
  timeout 900 python tools/calibrate.py $W gpurun_out/calib_${W}.json > gpurun_out/${TAG}_calib_${W}.txt 2>&1; echo "calib $W rc=$?"
done
du -sh gpurun_out
