set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02o_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02o_pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02o_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02o_smoke.txt
for W in vgg16 resnet18 wide_mlp mlp784 lenet5; do
  timeout 900 python bench.py --workload $W > gpurun_out/r02o_bench_${W}.json 2> gpurun_out/r02o_bench_${W}.err; echo "bench $W rc=$?"
  timeout 900 python bench.py --workload $W --impl reference > gpurun_out/r02o_ref_${W}.json 2>&1; echo "ref $W rc=$?"
done
