#!/bin/bash
# conv1 forward with the epilogue dropped (DEV timing probe PPB_GEMM_DBG=4):
# what bounds the K = 32 mainloop (67 MB of im2col rows in ~39 us)?
set -u
TAG=r02zi
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
PPB_GEMM_DBG=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 0 -c 1 -o gpurun_out/${TAG}_fwd1_noepi python tools/profile_ops.py vgg16 > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_fwd1_noepi.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_fwd1_noepi_source.csv 2>&1
ncu -i gpurun_out/${TAG}_fwd1_noepi.ncu-rep --page details --csv > gpurun_out/${TAG}_fwd1_noepi_details.csv 2>&1
ncu -i gpurun_out/${TAG}_fwd1_noepi.ncu-rep --page raw --csv > gpurun_out/${TAG}_fwd1_noepi_raw.csv 2>&1
rm -f gpurun_out/${TAG}_fwd1_noepi.ncu-rep
