set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
PPB_WGRAD_STREAMS2=1 timeout 900 python -m pytest tests/test_bench_parity_gpu.py tests/test_cnn_gpu.py -q -x -k "vgg16_b512_bench_config or lenet or small" > gpurun_out/r02r_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02r_tests.txt
for rep in 1 2 3; do
for v in "base" "PPB_WGRAD_STREAMS2=1"; do
  line=$(env $([ "$v" = base ] || echo $v) timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" "$rep $v" "$line"
done; done
PPB_WGRAD_STREAMS2=1 timeout 300 python tools/overlap_trace.py vgg16 1 stash_all > gpurun_out/r02r_timeline_2su.jsonl 2>&1
tail -1 gpurun_out/r02r_timeline_2su.jsonl | cut -c1-300
