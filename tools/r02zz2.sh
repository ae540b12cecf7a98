#!/bin/bash
# Batched bias-partial sums (side job, split-K bias job, bias_update_cols):
# parity, then VGG-16 / ResNet-18 timing and the per-op VGG-16 table vs r02zzf.
set -u
TAG=${TAG:-r02zz2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_resnet_gpu.py tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_cnn_gpu.py tests/test_bench_parity_gpu.py tests/test_train_gpu.py -q -x > gpurun_out/${TAG}_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.txt
for rep in 1 2 3; do
  line=$(timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('vgg', round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['roofline']['frac'])" "$line"
done
line=$(timeout 300 python bench.py --workload resnet18 --no-cpu-baseline --steps 50 2>/dev/null | tail -1)
python -c "import json,sys; d=json.loads(sys.argv[1]); print('resnet', round(d['ms_per_step'],4), round(d['value']), d['clocks']['sm_mhz'])" "$line"
timeout 300 python tools/profile_ops.py vgg16 > gpurun_out/${TAG}_ops_vgg16.jsonl 2>&1
python - <<'PY'
import json, os
tag = os.environ.get('TAG', 'r02zz2')
def load(f):
    d = {}
    for l in open(f):
        if l.startswith('{"kind"'):
            r = json.loads(l); k = (r['layer'], r['kind']); d[k] = d.get(k, 0) + r['ms']
    return d
a = load('profiles/r02/r02zzf_ops_vgg16.jsonl'); b = load('gpurun_out/' + tag + '_ops_vgg16.jsonl')
print('total', round(sum(a.values()) * 1000, 1), round(sum(b.values()) * 1000, 1))
for k in sorted(set(a) | set(b)):
    if abs(a.get(k, 0) - b.get(k, 0)) * 1000 > 3: print(k, round(a.get(k, 0) * 1000, 1), round(b.get(k, 0) * 1000, 1))
PY
