set -u
mkdir -p gpurun_out
timeout 300 python tools/mma_probe.py 3 > gpurun_out/r02g_mma_probe3.jsonl 2>&1; echo "probe2 rc=$?"; cat gpurun_out/r02g_mma_probe3.jsonl
