// Pieces shared by the tcgen05 kernels (gemm_tc.cu, conv_halo.cu): tile
// constants and the per-stage TMA operand loads.
#pragma once

#include <cuda.h>

#include "gemm.h"
#include "ptx.cuh"

namespace ppb {

constexpr int kBM = 128;  // rows of A per CTA
constexpr int kBK = 32;   // K per pipeline stage (one 128-byte swizzle row of fp32)

// TMA loads of one operand for one pipeline stage: `rows` MN-rows starting at
// mn0 (this CTA's slice) for K block kb.  CG = 2 signals the leader's barrier.
template <int CG>
struct Tma {
    uint64_t* bar;
    uint32_t bar_c;
    __device__ __forceinline__ void d2(void* dst, const CUtensorMap* m, int a, int b) const {
        if (CG == 2) tma_load_2d_pair(dst, m, bar_c, a, b);
        else tma_load_2d(dst, m, bar, a, b);
    }
    __device__ __forceinline__ void d3(void* dst, const CUtensorMap* m, int a, int b, int c) const {
        if (CG == 2) tma_load_3d_pair(dst, m, bar_c, a, b, c);
        else tma_load_3d(dst, m, bar, a, b, c);
    }
    __device__ __forceinline__ void d4(void* dst, const CUtensorMap* m, int a, int b, int c, int d) const {
        if (CG == 2) tma_load_4d_pair(dst, m, bar_c, a, b, c, d);
        else tma_load_4d(dst, m, bar, a, b, c, d);
    }
};

template <bool MN, int ROWS, int CG>
__device__ __forceinline__ void load_operand(const Tma<CG>& t, const CUtensorMap* map, const ConvGeom& g,
                                             uint8_t* dst, int mn0, int kb) {
    const int k0 = kb * kBK;
    if (g.mode == OP_DENSE) {
        if (MN) {
#pragma unroll
            for (int i = 0; i < ROWS / 32; ++i) t.d2(dst + i * 4096, map, mn0 + 32 * i, k0);
        } else {
            t.d2(dst, map, k0, mn0);
        }
    } else if (g.mode == OP_CONV_ROWS) {
        // 128 output pixels (rows) x 32 channels of tap t, channel block cb
        const int tap = kb / g.cblocks, cb = kb - tap * g.cblocks;
        const int r = tap / g.ksz, s = tap - r * g.ksz;
        const int img = mn0 / g.howo, rem = mn0 - img * g.howo, h0 = rem / g.wo;
        t.d4(dst, map, cb * 32, s + g.off, h0 + r + g.off, img);
    } else if (g.mode == OP_CONV_KPIX) {
        // 32 output pixels (K rows) x 32 channels per box; tap from the column
        const int p0 = k0;
        const int img = p0 / g.howo, rem = p0 - img * g.howo, h0 = rem / g.wo;
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) {
            const int col = mn0 + 32 * i;
            const int tap = col / g.ck, c0 = col - tap * g.ck;
            const int r = tap / g.ksz, s = tap - r * g.ksz;
            t.d4(dst + i * 4096, map, c0, s + g.off, h0 + r + g.off, img);
        }
    } else {  // OP_WFLIP
        const int tap = kb / g.cblocks, kblk = kb - tap * g.cblocks;
        const int tf = g.ksz * g.ksz - 1 - tap;
#pragma unroll
        for (int i = 0; i < ROWS / 32; ++i) t.d3(dst + i * 4096, map, mn0 + 32 * i, tf, kblk * 32);
    }
}

}  // namespace ppb
