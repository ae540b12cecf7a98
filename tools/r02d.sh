set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:halo_conv_kernel -s 2 -c 1 -o gpurun_out/r02d_conv2_dgrad $B > gpurun_out/r02d_n1.txt 2>&1; echo "ncu1 rc=$?"
timeout 600 $N -k regex:tc_gemm_kernel -s 1 -c 1 -o gpurun_out/r02d_conv2_fwd $B > gpurun_out/r02d_n2.txt 2>&1; echo "ncu2 rc=$?"
timeout 600 $N -k regex:tc_gemm_kernel -s 36 -c 1 -o gpurun_out/r02d_conv2_wgrad $B > gpurun_out/r02d_n3.txt 2>&1; echo "ncu3 rc=$?"
timeout 600 $N -k regex:tc_gemm_kernel -s 3 -c 1 -o gpurun_out/r02d_conv6_fwd $B > gpurun_out/r02d_n4.txt 2>&1; echo "ncu4 rc=$?"
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/r02d_n1.txt
