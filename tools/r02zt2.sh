#!/bin/bash
# Source-level stall sampling of VGG conv1's weight gradient (148-way split-K
# over pixels; last op of the backward, so its tail is on the step's critical path).
set -u
TAG=r02zt
mkdir -p gpurun_out
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$2" -s $3 -c 1 -o gpurun_out/${TAG}_$1 python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_source.csv 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>&1
  rm -f gpurun_out/${TAG}_$1.ncu-rep
  python tools/stall_summary.py gpurun_out/${TAG}_$1_source.csv 30 > gpurun_out/${TAG}_$1_stalls.txt 2>&1
  rm -f gpurun_out/${TAG}_$1_source.csv
}
run wgrad1 "tc_gemm_kernel<.*64, \(int\)1>" 0
grep -E "Duration|DRAM Throughput|Grid Size|Stages|Shared Memory Configuration Size|Registers" gpurun_out/${TAG}_wgrad1_details.csv | head -12
