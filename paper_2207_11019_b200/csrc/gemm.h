// Shard GEMM interface shared by the tcgen05 kernel (gemm_tc.cu), the exact
// fp32 SIMT kernel (gemm_simt.cu) and the executor.
//
//   C[m][n] = sum_k A(m,k) * B(n,k)          (fp32 accumulate)
//
// A(m,k) lives at a[m*lda + k] (K-major) or a[k*lda + m] (MN-major); the same
// for B with n in place of m.  The three products of the partitioned step map
// onto it as (reference tinynet.cpp:11-48, train_partitioned.cpp:281,505,515):
//
//   forward  q  = X . W_s^T     A = X  (K-major)  B = W_s (K-major)
//   dgrad    P  = d . W_s       A = d  (K-major)  B = W_s (MN-major)
//   wgrad    dW = d^T . X       A = d  (MN-major) B = X   (MN-major)
//
// The epilogue is where the partitioned step's neighbours are fused: bias +
// activation, the forward all-gather (multi-destination stores into every
// consumer's full-activation buffer), the backward scatter of partial input
// gradients into per-destination slots, the ReLU mask when the reduction is
// trivial, and the SGD update of the weight shard.
#pragma once

#include <cstdint>

namespace ppb {

enum EpiMode : int {
    EPI_STORE = 0,  // out = act(acc + bias[n]) stored to every dst[d]
    EPI_MASK = 1,   // out = acc * (mask[m][mcol0+n] > 0) stored to dst[0]
    EPI_SGD = 2,    // W[m][n] -= alpha * (acc * inv_b); non-finite acc -> *flag = 1
    EPI_SLOTS = 3,  // column segment s of acc stored to seg_dst[s] (backward scatter)
};

constexpr int kMaxDst = 8;

struct EpiParams {
    int mode = EPI_STORE;
    int M = 0, N = 0;  // valid extent of C
    // EPI_STORE / EPI_MASK: C(m,n) -> dst[d][m*ldd + col0 + n]
    float* dst[kMaxDst] = {};
    int ndst = 0;
    long long ldd = 0;
    int col0 = 0;
    const float* bias = nullptr;  // indexed by n, optional
    int relu = 0;
    // EPI_MASK
    const float* mask = nullptr;
    long long ldm = 0;
    int mcol0 = 0;
    // EPI_SGD
    float* W = nullptr;
    long long ldw = 0;
    const double* alpha = nullptr;  // device scalar (the reference keeps alpha in double)
    float inv_b = 1.f;
    int* flag = nullptr;
    // EPI_SLOTS: n in [seg_lo[s], seg_hi[s]) -> seg_dst[s][m*seg_ld[s] + n - seg_lo[s]],
    // optionally ReLU-masked by seg_mask[s][m*seg_mask_ld[s] + n] > 0 (used when
    // a layer has a single contributor, so the backward merge is a pure scatter).
    int nseg = 0;
    int seg_lo[kMaxDst] = {};
    int seg_hi[kMaxDst] = {};
    float* seg_dst[kMaxDst] = {};
    long long seg_ld[kMaxDst] = {};
    const float* seg_mask[kMaxDst] = {};
    long long seg_mask_ld[kMaxDst] = {};
};

// Host-side description of one operand: a row-major fp32 matrix of `rows` x
// `cols` with leading dimension `ld` (elements).  For a K-major operand rows is
// the M (or N) extent and cols is K; for an MN-major operand rows is K.
struct Operand {
    const float* ptr = nullptr;
    int rows = 0;
    int cols = 0;
    long long ld = 0;
    bool mn_major = false;
};

struct GemmDesc {
    Operand a, b;
    int M = 0, N = 0, K = 0;
    EpiParams epi;
};

}  // namespace ppb
