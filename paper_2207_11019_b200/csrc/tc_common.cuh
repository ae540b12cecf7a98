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

// Incremental per-tile operand addressing for the sequential K loop of
// tc_gemm_kernel: the divisions that map a K block / MN offset to (tap,
// channel block, image, row) happen once per tile in init(); advance() steps
// one K block with adds and compares only.  The TMA producer is a single
// thread, so per-box integer divisions (~25 instructions each) were its
// bottleneck on the conv wgrad shapes (6 boxes per K block).
template <bool MN, int ROWS, int CG>
struct OperandCursor {
    int a0, a1, a2;      // mode-dependent K-block state
    int img, h0;         // CONV_ROWS: tile pixel origin; KPIX: K-block pixel origin
    int cs[ROWS / 32];   // KPIX: per 32-column group: channel origin
    int cw[ROWS / 32];   //        column tap offset (s + off)
    int ch[ROWS / 32];   //        row tap offset (r + off)

    __device__ __forceinline__ void init(const ConvGeom& g, int mn0, int kb0) {
        if (g.mode == OP_CONV_ROWS || g.mode == OP_WFLIP) {
            const int tap = kb0 / g.cblocks;
            a0 = kb0 - tap * g.cblocks;  // channel block
            a1 = tap / g.ksz;            // r (ROWS) / tap (WFLIP uses a2)
            a2 = tap - a1 * g.ksz;       // s
            if (g.mode == OP_WFLIP) a1 = tap;
            if (g.mode == OP_CONV_ROWS) {
                img = mn0 / g.howo;
                h0 = (mn0 - img * g.howo) / g.wo;
            }
        } else if (g.mode == OP_CONV_KPIX) {
            const int p0 = kb0 * kBK;
            img = p0 / g.howo;
            h0 = (p0 - img * g.howo) / g.wo;
#pragma unroll
            for (int i = 0; i < ROWS / 32; ++i) {
                const int col = mn0 + 32 * i;
                const int tap = col / g.ck;
                const int r = tap / g.ksz;
                cs[i] = col - tap * g.ck;
                cw[i] = tap - r * g.ksz + g.off;
                ch[i] = r + g.off;
            }
        } else {
            a0 = kb0 * kBK;  // dense: k0
        }
    }

    __device__ __forceinline__ void load(const Tma<CG>& t, const CUtensorMap* map, const ConvGeom& g, uint8_t* dst,
                                         int mn0) const {
        if (g.mode == OP_DENSE) {
            if (MN) {
#pragma unroll
                for (int i = 0; i < ROWS / 32; ++i) t.d2(dst + i * 4096, map, mn0 + 32 * i, a0);
            } else {
                t.d2(dst, map, a0, mn0);
            }
        } else if (g.mode == OP_CONV_ROWS) {
            t.d4(dst, map, a0 * 32, a2 + g.off, h0 + a1 + g.off, img);
        } else if (g.mode == OP_CONV_KPIX) {
#pragma unroll
            for (int i = 0; i < ROWS / 32; ++i) t.d4(dst + i * 4096, map, cs[i], cw[i], h0 + ch[i], img);
        } else {  // OP_WFLIP
            const int tf = g.ksz * g.ksz - 1 - a1;
#pragma unroll
            for (int i = 0; i < ROWS / 32; ++i) t.d3(dst + i * 4096, map, mn0 + 32 * i, tf, a0 * 32);
        }
    }

    __device__ __forceinline__ void advance(const ConvGeom& g) {
        if (g.mode == OP_DENSE) {
            a0 += kBK;
        } else if (g.mode == OP_CONV_ROWS) {
            if (++a0 == g.cblocks) {
                a0 = 0;
                if (++a2 == g.ksz) {
                    a2 = 0;
                    ++a1;
                }
            }
        } else if (g.mode == OP_CONV_KPIX) {
            // 32 pixels per K block: whole rows of one image, or whole images
            if (g.howo >= kBK) {
                h0 += g.krows;
                if (h0 >= g.ho) {
                    h0 = 0;
                    ++img;
                }
            } else {
                img += g.kimgs;
            }
        } else {  // OP_WFLIP
            if (++a0 == g.cblocks) {
                a0 = 0;
                ++a1;
            }
        }
    }
};

}  // namespace ppb
