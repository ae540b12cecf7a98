#!/bin/bash
# Source-level stall sampling of the narrow conv2 kernels (halo dgrad, rank-4
# fwd, wgrad): per-SASS-instruction warp-stall reasons, exported to CSV on the box.
set -u
TAG=r02za
mkdir -p gpurun_out
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o gpurun_out/${TAG}_$1 python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_source.csv 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>&1
  rm -f gpurun_out/${TAG}_$1.ncu-rep
}
run halo_dgrad2 halo_conv 2
run fwd2 tc_gemm 1
ls -la gpurun_out | grep $TAG
