#!/bin/bash
# Tile / row-reuse sweep for conv3 dgrad (131072 x 64 x 1152), conv4 dgrad
# (131072 x 128 x 1152) and conv2 wgrad (576 x 64 x 524288) (DEV build knobs).
set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
i=0
run() {
  i=$((i+1))
  env "$@" timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/r02zj_ops_$i.jsonl 2>&1
  python - "$i" "$*" <<'PY'
import json, sys
rows=[json.loads(l) for l in open(f"gpurun_out/r02zj_ops_{sys.argv[1]}.jsonl") if l.startswith('{"kind"')]
sel=[(r['layer'], r['kind'][:5], r['bn'], r['cg'], r['splits'], r['halo'], round(r['ms']*1000,1)) for r in rows if (r['layer'] in (3,4) and r['kind']=='dgrad_gemm') or (r['layer']==2 and r['kind']!='pool_relayout')]
print(sys.argv[2], round(sum(r['ms'] for r in rows)*1000,1), sel)
PY
}
run X=1
run PPB_NO_ROW_REUSE=1
run PPB_FORCE_TILE="131072,64,1152,1,64,0;131072,128,1152,1,128,0"
run PPB_FORCE_TILE="576,64,524288,2,64,0"
run PPB_FORCE_TILE="576,64,524288,2,64,58"
run PPB_FORCE_TILE="576,64,524288,1,64,58"
run PPB_FORCE_TILE="576,64,524288,1,64,15"
