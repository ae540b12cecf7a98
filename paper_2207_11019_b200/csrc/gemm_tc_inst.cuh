// One (A_MN, B_MN) operand-major combination of the tcgen05 GEMM kernel:
// its six (BN, CG) instantiations, their launch and smem-attribute setup.
// Included by gemm_tc_inst_{ff,ft,tf,tt}.cu with PPB_A_MN / PPB_B_MN set.
#include "gemm_tc_kernel.cuh"

namespace ppb {

template <>
cudaError_t tc_launch_mn<PPB_A_MN, PPB_B_MN>(const TcGemmPlan& p, cudaStream_t s) {
    if (p.cg == 2) {
        switch (p.bn) {
            case 64: return launch_t<PPB_A_MN, PPB_B_MN, 64, 2>(p, s);
            case 128: return launch_t<PPB_A_MN, PPB_B_MN, 128, 2>(p, s);
            default: return launch_t<PPB_A_MN, PPB_B_MN, 256, 2>(p, s);
        }
    }
    switch (p.bn) {
        case 64: return launch_t<PPB_A_MN, PPB_B_MN, 64, 1>(p, s);
        case 128: return launch_t<PPB_A_MN, PPB_B_MN, 128, 1>(p, s);
        default: return launch_t<PPB_A_MN, PPB_B_MN, 256, 1>(p, s);
    }
}

template <>
cudaError_t tc_init_mn<PPB_A_MN, PPB_B_MN>() {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto kernel) {
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    };
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 64, 1>);
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 128, 1>);
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 256, 1>);
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 64, 2>);
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 128, 2>);
    set(tc_gemm_kernel<PPB_A_MN, PPB_B_MN, 256, 2>);
    return e;
}

}  // namespace ppb
