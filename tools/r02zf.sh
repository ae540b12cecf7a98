#!/bin/bash
# Source-level stall sampling: conv1 fwd (K = 32 im2col GEMM), conv3 dgrad
# (pooled merge), conv1 wgrad (148-way split-K).
set -u
TAG=r02zf
mkdir -p gpurun_out
run() {  # name regex skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o gpurun_out/${TAG}_$1 python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_source.csv 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>&1
  rm -f gpurun_out/${TAG}_$1.ncu-rep
}
run fwd1 tc_gemm 0
run dgrad3 tc_gemm 23
run wgrad1 tc_gemm 37
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/${TAG}_list.csv python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "list rc=$?"
ls -la gpurun_out | grep $TAG
