#!/bin/bash
# Single-thread MMA issue loop with incremental descriptors: parity + timing.
set -u
TAG=${TAG:-r02zb}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_cnn_gpu.py tests/test_bench_parity_gpu.py tests/test_resnet_gpu.py -q -x > gpurun_out/${TAG}_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.txt
for rep in 1 2; do
  line=$(timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('vgg', round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['roofline']['frac'])" "$line"
done
line=$(timeout 300 python bench.py --workload resnet18 --no-cpu-baseline --steps 50 2>/dev/null | tail -1)
python -c "import json,sys; d=json.loads(sys.argv[1]); print('resnet', round(d['ms_per_step'],4), d['value'])" "$line"
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/${TAG}_ops_vgg16.jsonl 2>&1
timeout 300 python tools/profile_ops.py resnet18 > gpurun_out/${TAG}_ops_resnet18.jsonl 2>&1
TAG=$TAG python - <<'PY'
import json
def load(f):
    d={}
    for l in open(f):
        if l.startswith('{"kind"'):
            r=json.loads(l); d[(r['layer'],r['kind'])]=d.get((r['layer'],r['kind']),0)+r['ms']
    return d
a=load('profiles/r02/r02zh_ops_vgg16.jsonl'); import os; b=load('gpurun_out/'+os.environ.get('TAG','r02zb')+'_ops_vgg16.jsonl')
print('total', round(sum(a.values())*1000,1), round(sum(b.values())*1000,1))
for k in sorted(a):
    if abs(a[k]-b.get(k,0))*1000 > 2: print(k, round(a[k]*1000,1), round(b.get(k,0)*1000,1))
PY
