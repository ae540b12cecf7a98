// Implicit-GEMM descriptors for a stride-1 k x k convolution over padded NHWC
// tensors (forward, dgrad, wgrad).  Shapes:
//   x_pad  [N][H+2p][W+2p][ldx]   input, zero border of p, channels [0, C)
//   w      [u][k*k][ck]           shard weights in GEMM layout (ck = C rounded
//                                 up to 32, zero-padded per tap), pitch k*k*ck
//   d_pad  [N][Ho+2q][Wo+2q][ldd] error signal of the shard (u channels),
//                                 zero border q = k-1-p, Ho = H+2p-k+1
// forward : q[N*Ho*Wo x u]   = sum_{tap,c} x_pad(pixel shifted by tap, c) w[u][tap][c]
// dgrad   : dx[N*H*W x C]    = sum_{tap,k} d_pad(pixel shifted by tap, k) w[k][flip(tap)][c]
// wgrad   : dw[u x k*k*ck]   = sum_{pixel}  d_pad(pixel + q, k) x_pad(pixel shifted by tap, c)
#pragma once

#include <utility>

#include "gemm.h"

namespace ppb {

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Spatial TMA box covering `pixels` consecutive output pixels of an ho x wo
// grid (whole rows, whole images).  False if the grid does not tile.
inline bool conv_box(int ho, int wo, int pixels, ConvGeom& g) {
    if (wo > 256 || ho < 1 || wo < 1) return false;
    const int hw = ho * wo;
    if (hw >= pixels) {
        if (pixels % wo != 0) return false;
        const int rows = pixels / wo;
        if (ho % rows != 0 || rows > 256) return false;
        g.bw = wo;
        g.bh = rows;
        g.bn = 1;
    } else {
        if (pixels % hw != 0) return false;
        g.bw = wo;
        g.bh = ho;
        g.bn = pixels / hw;
        if (g.bn > 256 || ho > 256) return false;
    }
    g.wo = wo;
    g.howo = hw;
    g.ho = ho;
    g.krows = hw >= 32 && 32 % wo == 0 ? 32 / wo : 1;
    g.kimgs = hw < 32 && 32 % hw == 0 ? 32 / hw : 1;
    return true;
}

struct ConvShape {
    int N = 0, H = 0, W = 0, C = 0;  // input
    int ksz = 3, pad = 1;
    int u = 0;                        // output channels of the shard
    int Ho() const { return H + 2 * pad - ksz + 1; }
    int Wo() const { return W + 2 * pad - ksz + 1; }
    int ck() const { return round_up(C, 32); }
    int q() const { return ksz - 1 - pad; }
};

// Implicit GEMM applies when the output grid tiles into 128-pixel (forward)
// and 32-pixel (wgrad) boxes and the input grid into 128-pixel boxes (dgrad).
inline bool conv_implicit_ok(const ConvShape& s) {
    ConvGeom g;
    return conv_box(s.Ho(), s.Wo(), 128, g) && conv_box(s.Ho(), s.Wo(), 32, g) && conv_box(s.H, s.W, 128, g);
}

inline GemmDesc conv_fwd_desc(const ConvShape& s, const float* x_pad, long long ldx, const float* w) {
    GemmDesc d;
    d.a.ptr = x_pad;
    d.a.mn_major = false;
    d.a.ld = ldx;
    d.a.ch = s.C;
    d.a.wp = s.W + 2 * s.pad;
    d.a.hp = s.H + 2 * s.pad;
    d.a.imgs = s.N;
    conv_box(s.Ho(), s.Wo(), 128, d.a.geom);
    d.a.geom.mode = OP_CONV_ROWS;
    d.a.geom.ksz = s.ksz;
    d.a.geom.cblocks = s.ck() / 32;
    d.a.geom.off = 0;
    const int K = s.ksz * s.ksz * s.ck();
    d.b = Operand{w, s.u, K, K, false};
    d.M = s.N * s.Ho() * s.Wo();
    d.N = s.u;
    d.K = K;
    return d;
}

inline GemmDesc conv_dgrad_desc(const ConvShape& s, const float* d_pad, long long ldd, const float* w) {
    GemmDesc d;
    const int q = s.q();
    d.a.ptr = d_pad;
    d.a.mn_major = false;
    d.a.ld = ldd;
    d.a.ch = s.u;
    d.a.wp = s.Wo() + 2 * q;
    d.a.hp = s.Ho() + 2 * q;
    d.a.imgs = s.N;
    conv_box(s.H, s.W, 128, d.a.geom);  // rows = input pixels
    d.a.geom.mode = OP_CONV_ROWS;
    d.a.geom.ksz = s.ksz;
    d.a.geom.cblocks = round_up(s.u, 32) / 32;
    d.a.geom.off = 0;
    const int ck = s.ck();
    d.b.ptr = w;
    d.b.mn_major = true;
    d.b.ld = ck;
    d.b.ch = ck;
    d.b.wp = s.ksz * s.ksz;
    d.b.hp = s.u;
    d.b.imgs = 1;
    d.b.geom.mode = OP_WFLIP;
    d.b.geom.ksz = s.ksz;
    d.b.geom.cblocks = d.a.geom.cblocks;
    d.M = s.N * s.H * s.W;
    d.N = s.C;
    d.K = s.ksz * s.ksz * d.a.geom.cblocks * 32;
    return d;
}

// transposed = true computes dW^T (M = k*k*ck, N = u): better tile occupancy
// when u < 128; pair it with EpiParams::sgd_t.
inline GemmDesc conv_wgrad_desc(const ConvShape& s, const float* d_pad, long long ldd, const float* x_pad,
                                long long ldx, bool transposed = false) {
    GemmDesc d;
    const int q = s.q();
    d.a.ptr = d_pad;
    d.a.mn_major = true;
    d.a.ld = ldd;
    d.a.ch = s.u;
    d.a.wp = s.Wo() + 2 * q;
    d.a.hp = s.Ho() + 2 * q;
    d.a.imgs = s.N;
    conv_box(s.Ho(), s.Wo(), 32, d.a.geom);
    d.a.geom.mode = OP_CONV_KPIX;
    d.a.geom.ksz = 1;
    d.a.geom.ck = 1 << 30;  // one "tap": column = channel
    d.a.geom.off = q;
    d.b.ptr = x_pad;
    d.b.mn_major = true;
    d.b.ld = ldx;
    d.b.ch = s.C;
    d.b.wp = s.W + 2 * s.pad;
    d.b.hp = s.H + 2 * s.pad;
    d.b.imgs = s.N;
    conv_box(s.Ho(), s.Wo(), 32, d.b.geom);
    d.b.geom.mode = OP_CONV_KPIX;
    d.b.geom.ksz = s.ksz;
    d.b.geom.ck = s.ck();
    d.b.geom.off = 0;
    d.M = s.u;
    d.N = s.ksz * s.ksz * s.ck();
    d.K = s.N * s.Ho() * s.Wo();
    if (transposed) {
        std::swap(d.a, d.b);
        std::swap(d.M, d.N);
    }
    return d;
}

}  // namespace ppb
