set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dropin_gpu.py -q -x > gpurun_out/r02b_dropin.txt 2>&1; echo "dropin rc=$?"; tail -2 gpurun_out/r02b_dropin.txt
timeout 300 python tools/mma_probe.py > gpurun_out/r02b_mma_probe.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/r02b_mma_probe.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"halo_conv_kernel<1, 64" -s 0 -c 1 -o gpurun_out/r02b_conv2_dgrad python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel<0, 0, 64, 2>" -s 1 -c 1 -o gpurun_out/r02b_conv2_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel<1, 1, 64, 1>" -s 0 -c 2 -o gpurun_out/r02b_wgrad64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel<0, 0, 256, 2>" -s 0 -c 3 -o gpurun_out/r02b_bn256 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu4 rc=$?"
ls -la gpurun_out/*.ncu-rep
