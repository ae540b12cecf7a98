set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
timeout 600 python -m pytest tests/test_conv_gpu.py tests/test_cnn_gpu.py -q -x > gpurun_out/r02p_conv.txt 2>&1; echo "conv rc=$?"; tail -1 gpurun_out/r02p_conv.txt
for rep in 1 2; do
for v in "base" "PPB_NO_MASK_DBUF=1" "PPB_NO_MASK_PREFETCH=1 PPB_NO_MASK_DBUF=1"; do
  env $([ "$v" = base ] || echo $v) timeout 300 python tools/profile_ops.py vgg16 > "gpurun_out/r02p_ops_${rep}_${v// /_}.jsonl" 2>&1
  line=$(env $([ "$v" = base ] || echo $v) timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" "$rep $v" "$line"
done; done
