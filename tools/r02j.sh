set -u
mkdir -p gpurun_out
export PPB_LIB_PATH=$PWD/paper_2207_11019_b200/libpipeplan_b200_dev.so
for v in "base" "PPB_HALO_DBG=8" "PPB_HALO_DBG=4" "PPB_HALO_DBG=12" "PPB_HALO_DBG=14" "PPB_HALO_ALWAYS=1" "PPB_HALO_ALWAYS=1 PPB_HALO_DBG=8" "PPB_HALO_ALWAYS=1 PPB_HALO_DBG=12"; do
  env $([ "$v" = base ] || echo $v) timeout 300 python tools/profile_ops.py vgg16 > "gpurun_out/r02j_ops_${v// /_}.jsonl" 2>&1; echo "$v rc=$?"
done
