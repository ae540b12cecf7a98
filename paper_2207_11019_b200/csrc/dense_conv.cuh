// Dense-conv weight update for 3x3 / pad 1 on a 2x2 grid (kernels.cu
// dense_conv_update_2x2_kernel and the GEMM side job share it): one (co, ci)
// pair folds its 16 dWx entries onto the 9 taps in ascending (p, q) order,
// applies SGD to W and rewrites the 16 Wx entries.
#pragma once

#include "kernels.h"

namespace ppb {

__device__ __forceinline__ void dense_conv_update_2x2_item(const DenseConvGeom& g, const float* __restrict__ dWx,
                                                           float* __restrict__ W, float* __restrict__ Wx, float a,
                                                           float inv_b, int* flag, long long i) {
    const int co = static_cast<int>(i / g.C), ci = static_cast<int>(i % g.C);
    float v[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[p][q] = dWx[static_cast<long long>(p * g.u + co) * g.ldx + q * g.C + ci];
    float gs[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) gs[t] = 0.f;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) gs[((q >> 1) - (p >> 1) + 1) * 3 + ((q & 1) - (p & 1) + 1)] += v[p][q];
    bool bad = false;
    float wn[9];
    float* wr = W + co * g.ldw + ci;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const float gr = gs[t] * inv_b;
        bad |= !isfinite(gr);
        wn[t] = wr[t * g.ck] - a * gr;
        wr[t * g.ck] = wn[t];
    }
    if (bad && flag != nullptr) atomicOr(flag, 1);
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            Wx[static_cast<long long>(p * g.u + co) * g.ldx + q * g.C + ci] =
                wn[((q >> 1) - (p >> 1) + 1) * 3 + ((q & 1) - (p & 1) + 1)];
}

inline bool dense_conv_is_2x2(const DenseConvGeom& g) {
    return g.k == 3 && g.pad == 1 && g.H == 2 && g.W == 2 && g.Ho == 2 && g.Wo == 2;
}

}  // namespace ppb
