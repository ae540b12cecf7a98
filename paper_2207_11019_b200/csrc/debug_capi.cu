// Diagnostic C entry points (kernel-level unit tests).  Not part of the
// reference boundary; declared in include/pipeplan_b200.h under "diagnostics".
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "capi_common.h"
#include "gemm_tc.h"

using namespace ppb;

extern "C" int ppb_debug_gemm(const float* a, int a_rows, int a_cols, long long lda, int a_mn,
                              const float* b, int b_rows, int b_cols, long long ldb, int b_mn,
                              int M, int N, int K, int mode, float* c, long long ldc,
                              const float* bias, int relu, const float* mask, long long ldm,
                              const double* alpha, float inv_b, int* flag, int precision,
                              int force_bn, void* stream) {
    GemmDesc d;
    d.a = Operand{a, a_rows, a_cols, lda, a_mn != 0};
    d.b = Operand{b, b_rows, b_cols, ldb, b_mn != 0};
    d.M = M;
    d.N = N;
    d.K = K;
    d.epi.mode = mode;
    d.epi.dst[0] = c;
    d.epi.ndst = 1;
    d.epi.ldd = ldc;
    d.epi.bias = bias;
    d.epi.relu = relu;
    d.epi.mask = mask;
    d.epi.ldm = ldm;
    d.epi.W = c;
    d.epi.ldw = ldc;
    d.epi.alpha = alpha;
    d.epi.inv_b = inv_b;
    d.epi.flag = flag;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (precision == 1) {
        e = simt_gemm_launch(d, s);
    } else {
        TcGemmPlan p;
        char err[256];
        if (!tc_gemm_prepare(d, &p, force_bn, err, sizeof(err))) {
            ppb_set_error(err);
            return PPB_ERR_CUDA;
        }
        e = tc_gemm_launch(p, s);
    }
    if (e != cudaSuccess) {
        ppb_set_error(cudaGetErrorString(e));
        return PPB_ERR_CUDA;
    }
    return PPB_OK;
}
