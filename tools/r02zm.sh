#!/bin/bash
# ResNet-18 memory-bound kernels: shortcut add + ReLU fused into the GEMM
# epilogue (identity residual layers), no U write-back in residual_act,
# unrolled col2im (k = 3), two positions in flight in conv_merge_res.
# Parity first, then timing, per-op profile and ncu DRAM bytes of the
# elementwise kernels of the ResNet-18 step.
set -u
TAG=${TAG:-r02zm}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_resnet_gpu.py tests/test_gemm_gpu.py tests/test_conv_gpu.py tests/test_cnn_gpu.py tests/test_bench_parity_gpu.py -q -x > gpurun_out/${TAG}_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/${TAG}_tests.txt
for rep in 1 2; do
  line=$(timeout 300 python bench.py --workload resnet18 --no-cpu-baseline --steps 50 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('resnet', round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])" "$line"
done
line=$(timeout 300 python bench.py --no-cpu-baseline --steps 200 2>/dev/null | tail -1)
python -c "import json,sys; d=json.loads(sys.argv[1]); print('vgg', round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['roofline']['frac'])" "$line"
timeout 300 python tools/profile_ops.py resnet18 > gpurun_out/${TAG}_ops_resnet18.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'conv_merge|col2im|im2col|residual|pool_fwd' --clock-control none --csv --log-file gpurun_out/${TAG}_ew_resnet.csv python bench.py --workload resnet18 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ew rc=$?"
python tools/ew_ncu.py gpurun_out/${TAG}_ew_resnet.csv > gpurun_out/${TAG}_ew_resnet_summary.jsonl 2>&1
python - <<'PY'
import json, os
tag = os.environ.get('TAG', 'r02zm')
def load(f):
    d = {}
    for l in open(f):
        if l.startswith('{"kind"'):
            r = json.loads(l); k = (r['layer'], r['kind']); d[k] = d.get(k, 0) + r['ms']
    return d
a = load(os.environ.get('BASE', 'profiles/r02/r02zl_ops_resnet18.jsonl')); b = load('gpurun_out/' + tag + '_ops_resnet18.jsonl')
print('total', round(sum(a.values()) * 1000, 1), round(sum(b.values()) * 1000, 1))
for k in sorted(set(a) | set(b)):
    if abs(a.get(k, 0) - b.get(k, 0)) * 1000 > 5: print(k, round(a.get(k, 0) * 1000, 1), round(b.get(k, 0) * 1000, 1))
PY
