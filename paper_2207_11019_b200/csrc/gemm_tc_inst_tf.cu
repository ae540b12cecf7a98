#define PPB_A_MN true
#define PPB_B_MN false
#include "gemm_tc_inst.cuh"
