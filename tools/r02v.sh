set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
PPB_GEMM_DBG=16 PPB_HALO_DBG=16 timeout 900 python -m pytest tests/test_conv_gpu.py tests/test_cnn_gpu.py tests/test_bench_parity_gpu.py -q -x -k "not large_step and not microbatched and not teacher" > gpurun_out/r02v_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02v_tests.txt
for rep in 1 2 3; do for v in "base" "PPB_GEMM_DBG=16 PPB_HALO_DBG=16"; do
  line=$(env $([ "$v" = base ] || echo $v) timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" "$rep $v" "$line"
done; done
for v in "base" "PPB_GEMM_DBG=16 PPB_HALO_DBG=16"; do
  env $([ "$v" = base ] || echo $v) timeout 300 python tools/profile_ops.py vgg16 > "gpurun_out/r02v_ops_${v%% *}.jsonl" 2>&1
done
python - <<'PY'
import json
def load(f):
    d={}
    for l in open(f):
        if l.startswith('{"kind"'):
            r=json.loads(l); d[(r['layer'],r['kind'])]=d.get((r['layer'],r['kind']),0)+r['ms']
    return d
a=load('gpurun_out/r02v_ops_base.jsonl'); b=load('gpurun_out/r02v_ops_PPB_GEMM_DBG=16.jsonl')
print('total', round(sum(a.values())*1000,1), round(sum(b.values())*1000,1))
for k in sorted(a):
    if abs(a[k]-b.get(k,0))*1000 > 3: print(k, round(a[k]*1000,1), round(b.get(k,0)*1000,1))
PY
