set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
for v in "base" "PPB_WGRAD_PAIR=1"; do
  env $([ "$v" = base ] || echo $v) timeout 300 python tools/profile_ops.py vgg16 > "gpurun_out/r02t_ops_${v}.jsonl" 2>&1
done
for rep in 1 2; do for v in "base" "PPB_WGRAD_PAIR=1"; do
  line=$(env $([ "$v" = base ] || echo $v) timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" "$rep $v" "$line"
done; done
python - <<'PY'
import json
for v in ("base","PPB_WGRAD_PAIR=1"):
    rows=[json.loads(l) for l in open(f"gpurun_out/r02t_ops_{v}.jsonl") if l.startswith('{"kind"')]
    print(v, [(r['layer'], r['bn'], r['cg'], r['splits'], round(r['ms']*1000,1)) for r in rows if r['kind']=='wgrad_sgd_gemm' and r['layer']<=4])
PY
