#define PPB_A_MN false
#define PPB_B_MN true
#include "gemm_tc_inst.cuh"
