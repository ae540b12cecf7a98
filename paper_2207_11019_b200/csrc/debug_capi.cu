// Diagnostic C entry points (kernel-level unit tests).  Not part of the
// reference boundary; declared in include/pipeplan_b200.h under "diagnostics".
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "capi_common.h"
#include "gemm_tc.h"

using namespace ppb;

namespace {
// split-K workspace for the diagnostic entry points (grown, never freed)
float* debug_ws(size_t n) {
    static float* p[32] = {};
    static size_t cap[32] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (cap[dev & 31] < n) {
        if (p[dev & 31]) cudaFree(p[dev & 31]);
        if (cudaMalloc(&p[dev & 31], n * sizeof(float)) != cudaSuccess) return nullptr;
        cap[dev & 31] = n;
    }
    return p[dev & 31];
}
}  // namespace

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
        if (!tc_gemm_prepare(d, &p, force_bn, err, sizeof(err), force_bn == 0 ? WsAlloc(debug_ws) : WsAlloc())) {
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

// Implicit-GEMM convolution products on device pointers (kernel unit tests):
// which = 0 forward (out [N*Ho*Wo x ldo], cols u), 1 dgrad (out [N*H*W x ldo],
// cols C), 2 wgrad (out [u x ldo], cols k*k*ck).  Layouts: csrc/conv.h.
#include "conv.h"

extern "C" int ppb_debug_conv(int which, const float* x_pad, int N, int H, int W, int C, long long ldx, int pad,
                              int ksz, const float* w, int u, const float* d_pad, long long ldd, float* out,
                              long long ldo, int force_bn, void* stream) {
    ConvShape s;
    s.N = N;
    s.H = H;
    s.W = W;
    s.C = C;
    s.ksz = ksz;
    s.pad = pad;
    s.u = u;
    if (!conv_implicit_ok(s)) {
        ppb_set_error("conv geometry does not tile into TMA boxes");
        return PPB_ERR_INVALID_ARGUMENT;
    }
    // which = 3: wgrad in the transposed orientation (dW^T), stored as SGD
    // with alpha = 1 and inv_b = -1 onto out (zeroed by the caller) so that
    // out[u][k*k*ck] receives dW.
    GemmDesc d = which == 0 ? conv_fwd_desc(s, x_pad, ldx, w)
                 : which == 1 ? conv_dgrad_desc(s, d_pad, ldd, w)
                              : conv_wgrad_desc(s, d_pad, ldd, x_pad, ldx, which == 3);
    d.epi.mode = EPI_STORE;
    d.epi.dst[0] = out;
    d.epi.ndst = 1;
    d.epi.ldd = ldo;
    static double* one = nullptr;
    if (which == 3) {
        if (one == nullptr) {
            const double v = 1.0;
            cudaMalloc(&one, sizeof(double));
            cudaMemcpy(one, &v, sizeof(double), cudaMemcpyHostToDevice);
        }
        d.epi.mode = EPI_SGD;
        d.epi.W = out;
        d.epi.ldw = ldo;
        d.epi.sgd_t = 1;
        d.epi.alpha = one;
        d.epi.inv_b = -1.f;
    }
    TcGemmPlan p;
    char err[256];
    if (!tc_gemm_prepare(d, &p, force_bn, err, sizeof(err), force_bn == 0 ? WsAlloc(debug_ws) : WsAlloc())) {
        ppb_set_error(err);
        return PPB_ERR_CUDA;
    }
    cudaError_t e = tc_gemm_launch(p, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
        ppb_set_error(cudaGetErrorString(e));
        return PPB_ERR_CUDA;
    }
    return PPB_OK;
}
