set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
for v in "base" "PPB_GEMM_DBG=4 PPB_HALO_DBG=2" "PPB_GEMM_DBG=2 PPB_HALO_DBG=2" "PPB_GEMM_DBG=8"; do
  env $([ "$v" = base ] || echo $v) timeout 300 python tools/profile_ops.py vgg16 > "gpurun_out/r02h_ops_${v// /_}.jsonl" 2>&1; echo "$v rc=$?"
done
