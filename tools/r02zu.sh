#!/bin/bash
# Round-2 closing evidence after the residual-extension kernel work: full
# pytest -m gpu, smoke, bench lines (both arms) of every workload, ncu launch
# lists (VGG-16 and ResNet-18) and the elementwise HBM summaries.
set -u
TAG=${TAG:-r02zu}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
for W in vgg16 resnet18 wide_mlp mlp784 lenet5; do
  timeout 900 python bench.py --workload $W > gpurun_out/${TAG}_bench_${W}.json 2> /dev/null; echo "bench $W rc=$?"
  timeout 900 python bench.py --workload $W --impl reference > gpurun_out/${TAG}_ref_${W}.json 2>&1; echo "ref $W rc=$?"
done
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/${TAG}_ops_vgg16.jsonl 2>&1
timeout 300 python tools/profile_ops.py resnet18 > gpurun_out/${TAG}_ops_resnet18.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches_resnet18.csv python bench.py --workload resnet18 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list resnet rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'pool_fwd|conv_merge|dense_conv|splitk_epilogue|colsum|bias_update|loss_head|im2col|col2im|reduce_mask|finalize|residual' --clock-control none --csv --log-file gpurun_out/${TAG}_ew_resnet.csv python bench.py --workload resnet18 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/${TAG}_ew_resnet.csv > gpurun_out/${TAG}_ew_resnet_summary.jsonl
rm -f gpurun_out/${TAG}_ew_resnet.csv
du -sh gpurun_out
