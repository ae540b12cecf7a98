set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dropin_gpu.py -q -x > gpurun_out/r02c_dropin.txt 2>&1; echo "dropin rc=$?"; tail -2 gpurun_out/r02c_dropin.txt
timeout 300 python tools/mma_probe.py > gpurun_out/r02c_mma_probe.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/r02c_mma_probe.jsonl
