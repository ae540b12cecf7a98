#define PPB_A_MN false
#define PPB_B_MN false
#include "gemm_tc_inst.cuh"
