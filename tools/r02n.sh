set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_resnet_gpu.py -q -x -s > gpurun_out/r02n_resnet.txt 2>&1; echo "resnet rc=$?"; grep -E "n=|passed|failed|Error|error" gpurun_out/r02n_resnet.txt | head -20
timeout 600 python bench.py --workload resnet18 --no-cpu-baseline --steps 20 > gpurun_out/r02n_bench_resnet18.json 2> gpurun_out/r02n_bench_resnet18.err; echo "bench rc=$?"; tail -3 gpurun_out/r02n_bench_resnet18.err
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['step_tflops'], d['roofline']['per_kind_ms'])" gpurun_out/r02n_bench_resnet18.json
