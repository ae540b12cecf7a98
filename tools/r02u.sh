set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
S=512,2048,2048
i=0
for v in "" "$S,2,256,1" "$S,2,256,4" "$S,2,128,1" "$S,2,128,2" "$S,1,128,1" "$S,1,256,2" "$S,2,64,2"; do
  i=$((i+1))
  if [ -z "$v" ]; then timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/r02u_ops_$i.jsonl 2>&1
  else PPB_FORCE_TILE="$v" timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/r02u_ops_$i.jsonl 2>&1; fi
  python - "$i" "$v" <<'PY'
import json, sys
rows=[json.loads(l) for l in open(f"gpurun_out/r02u_ops_{sys.argv[1]}.jsonl") if l.startswith('{"kind"')]
sel=[(r['layer'], r['kind'][:5], r['bn'], r['cg'], r['splits'], round(r['ms']*1000,1)) for r in rows if r['layer'] in (11,12,13) and 'gemm' in r['kind'] and 'wgrad' not in r['kind']]
tot=sum(x[-1] for x in sel)
print(sys.argv[2] or 'auto', round(tot,1), sel)
PY
done
