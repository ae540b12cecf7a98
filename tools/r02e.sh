set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
N="ncu --set full --clock-control none --import-source on"
run() {  # name filter skip
  timeout 600 $N -k regex:$2 -s $3 -c 1 -o /tmp/$1 $B > /dev/null 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/r02e_$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/r02e_$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/r02e_$1_sass.csv 2>&1
  ls -la gpurun_out/r02e_$1_*
}
run conv2_dgrad halo_conv_kernel 2
run conv2_fwd tc_gemm_kernel 1
run conv2_wgrad tc_gemm_kernel 36
run conv6_fwd tc_gemm_kernel 3
du -sh gpurun_out
