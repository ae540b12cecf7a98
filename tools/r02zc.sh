#!/bin/bash
# Source-level stall sampling after the issue-loop change: halo conv2 dgrad,
# conv2 fwd (rank-4 implicit), conv2 wgrad (bn64, 1-CTA, split-K).
set -u
TAG=r02zc
mkdir -p gpurun_out
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 -o gpurun_out/${TAG}_$1 python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_source.csv 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>&1
  rm -f gpurun_out/${TAG}_$1.ncu-rep
}
run halo_dgrad2 halo_conv 2
run fwd2 tc_gemm 1
run wgrad2 "tc_gemm_kernel<.*64, \(int\)1>" 0
ls -la gpurun_out | grep $TAG
