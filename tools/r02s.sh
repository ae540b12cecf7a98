set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_bench_parity_gpu.py tests/test_cnn_gpu.py tests/test_train_gpu.py tests/test_resnet_gpu.py -q -x > gpurun_out/r02s_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02s_tests.txt
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
for rep in 1 2 3; do
for v in "base" "PPB_WGRAD_STRICT=1" "PPB_WGRAD_STRICT=1 PPB_WGRAD_ONE_STREAM=1"; do
  line=$(env $([ "$v" = base ] || echo $v) timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" "$rep $v" "$line"
done; done
timeout 300 python tools/overlap_trace.py vgg16 1 stash_all > gpurun_out/r02s_timeline.jsonl 2>&1
