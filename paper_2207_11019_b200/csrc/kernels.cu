// Non-GEMM kernels of the partitioned step.  All are HBM-bound (bytes per
// element listed per kernel in DESIGN.md) and deterministic: every reduction
// uses a fixed tree shape, never atomics on floating-point values.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "kernels.h"
#include "ptx.cuh"
#include "dense_conv.cuh"

namespace ppb {

namespace {
// Programmatic dependent launch for the step's small kernels (each calls
// griddep_wait() before touching its predecessor's results).
template <typename... P, typename... A>
cudaError_t pdl_launch(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}
}  // namespace

namespace {

constexpr int kRowThreads = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (value, index) max with first-index tie break.
__device__ __forceinline__ void argmax_merge(float& v, int& i, float ov, int oi) {
    if (ov > v || (ov == v && oi < i)) {
        v = ov;
        i = oi;
    }
}

template <int NT>
__device__ void block_argmax(float& v, int& i) {
    __shared__ float sv[NT / 32];
    __shared__ int si[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, i, o);
        argmax_merge(v, i, ov, oi);
    }
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) {
        sv[w] = v;
        si[w] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < NT / 32; ++k) argmax_merge(sv[0], si[0], sv[k], si[k]);
    }
    __syncthreads();
    v = sv[0];
    i = si[0];
    __syncthreads();
}

template <int NT>
__device__ float block_sum(float v) {
    __shared__ float s[NT / 32];
    v = warp_sum(v);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) s[w] = v;
    __syncthreads();
    float r = 0.f;
    if (threadIdx.x == 0) {
        for (int k = 0; k < NT / 32; ++k) r += s[k];
        s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}

template <int NT>
__device__ double block_sum_d(double v) {
    __shared__ double s[NT / 32];
    v = warp_sum_d(v);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) s[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        for (int k = 0; k < NT / 32; ++k) r += s[k];
        s[0] = r;
    }
    __syncthreads();
    r = s[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kRowThreads) loss_head_kernel(
    const float* __restrict__ in, long long ld_in, int F, const int* __restrict__ labels,
    int loss_kind, int relu_last, LossTargets t, double* __restrict__ loss_row,
    int* __restrict__ correct_row) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int row = blockIdx.x;
    const float* x = in + static_cast<long long>(row) * ld_in;
    const int label = labels[row];
    // argmax (prediction) over the row, first index on ties
    float bv = -FLT_MAX;
    int bi = 0x7fffffff;
    for (int c = threadIdx.x; c < F; c += kRowThreads) argmax_merge(bv, bi, x[c], c);
    block_argmax<kRowThreads>(bv, bi);

    if (loss_kind == 1) {
        // ---- softmax + cross entropy (tinynet.cpp:104-117, :232-238)
        const float mx = bv;
        float se = 0.f;
        for (int c = threadIdx.x; c < F; c += kRowThreads) se += expf(x[c] - mx);
        se = block_sum<kRowThreads>(se);
        const float inv = 1.f / se;
        for (int k = 0; k < t.n; ++k) {
            float* d = t.delta[k] + static_cast<long long>(row) * t.ld[k];
            for (int c = t.lo[k] + threadIdx.x; c < t.hi[k]; c += kRowThreads) {
                const float p = expf(x[c] - mx) * inv;
                d[c - t.lo[k]] = p - (c == label ? 1.f : 0.f);
            }
        }
        if (threadIdx.x == 0 && loss_row != nullptr) {
            // -log(max(p_label, 1e-300)) via log-sum-exp in double
            double l = static_cast<double>(mx) - static_cast<double>(x[label]) + log(static_cast<double>(se));
            const double cap = 690.77552789821368;  // -log(1e-300)
            loss_row[row] = l < cap ? l : cap;
            correct_row[row] = (F == 1 ? 1 : bi) == label;
        }
    } else {
        // ---- mse, 1/2 convention (tinynet.cpp:222-229, :275-279)
        double part = 0.0;
        for (int c = threadIdx.x; c < F; c += kRowThreads) {
            const float tg = F == 1 ? static_cast<float>(label) : (c == label ? 1.f : 0.f);
            const float d = x[c] - tg;
            part += 0.5 * static_cast<double>(d) * static_cast<double>(d);
        }
        for (int k = 0; k < t.n; ++k) {
            float* dd = t.delta[k] + static_cast<long long>(row) * t.ld[k];
            for (int c = t.lo[k] + threadIdx.x; c < t.hi[k]; c += kRowThreads) {
                const float tg = F == 1 ? static_cast<float>(label) : (c == label ? 1.f : 0.f);
                float d = x[c] - tg;
                if (relu_last && !(x[c] > 0.f)) d = 0.f;
                dd[c - t.lo[k]] = d;
            }
        }
        part = block_sum_d<kRowThreads>(part);
        if (threadIdx.x == 0 && loss_row != nullptr) {
            loss_row[row] = part;
            const int pred = F == 1 ? (x[0] >= 0.5f ? 1 : 0) : bi;
            correct_row[row] = pred == label;
        }
    }
}

__global__ void reduce_mask_kernel(ReduceSlots slots, long long ld_slot, int rows, int cols,
                                   const float* __restrict__ mask, long long ld_mask,
                                   float* __restrict__ out, long long ld_out, bool vec) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    if (vec) {
        const int c4 = cols / 4;
        const long long total = static_cast<long long>(rows) * c4;
        for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
             i += static_cast<long long>(gridDim.x) * blockDim.x) {
            const int r = static_cast<int>(i / c4), c = static_cast<int>(i % c4) * 4;
            float4 acc = *reinterpret_cast<const float4*>(slots.slot[0] + r * ld_slot + c);
            for (int k = 1; k < slots.n; ++k) {
                const float4 v = *reinterpret_cast<const float4*>(slots.slot[k] + r * ld_slot + c);
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            if (mask != nullptr) {
                const float4 m = *reinterpret_cast<const float4*>(mask + r * ld_mask + c);
                acc.x = m.x > 0.f ? acc.x : 0.f;
                acc.y = m.y > 0.f ? acc.y : 0.f;
                acc.z = m.z > 0.f ? acc.z : 0.f;
                acc.w = m.w > 0.f ? acc.w : 0.f;
            }
            *reinterpret_cast<float4*>(out + r * ld_out + c) = acc;
        }
        return;
    }
    const long long total = static_cast<long long>(rows) * cols;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
        float acc = slots.slot[0][r * ld_slot + c];
        for (int k = 1; k < slots.n; ++k) acc += slots.slot[k][r * ld_slot + c];
        if (mask != nullptr && !(mask[r * ld_mask + c] > 0.f)) acc = 0.f;
        out[r * ld_out + c] = acc;
    }
}

// Column sums of delta [rows x u] (pitch ld) into partial[blockIdx.x][u]:
// block b owns rows [b*per, (b+1)*per); thread = (channel group g of VEC
// channels, row lane j) with g fixed for the thread (blockDim % groups == 0),
// rows j, j+lanes, ... summed in ascending order, 4 loads in flight; then a
// fixed-order sum over the row lanes (deterministic).
template <int VEC>
__global__ void colsum_rows_kernel(const float* __restrict__ delta, long long ld, long long rows, int u,
                                   float* __restrict__ partial) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int groups = u / VEC;
    const int gpb = groups < 256 ? groups : 256;  // channel groups per block (blockIdx.y: group block)
    const int g = blockIdx.y * gpb + threadIdx.x % gpb, j = threadIdx.x / gpb;
    const int lanes = blockDim.x / gpb;
    const bool live = g < groups;
    const long long per = (rows + gridDim.x - 1) / gridDim.x;
    const long long r0 = blockIdx.x * per;
    const long long r1 = r0 + per < rows ? r0 + per : rows;
    const float* base = delta + g * VEC;
    float acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
    long long r = live ? r0 + j : r1;
    for (; r + 3LL * lanes < r1; r += 4LL * lanes) {
        float v[4][VEC];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float* p = base + (r + q * lanes) * ld;
            if (VEC == 4) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(p));
                v[q][0] = t.x; v[q][1] = t.y; v[q][2] = t.z; v[q][3] = t.w;
            } else {
                v[q][0] = __ldg(p);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc[k] += v[q][k];
    }
    for (; r < r1; r += lanes) {
        const float* p = base + r * ld;
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[k] += __ldg(p + k);
    }
    extern __shared__ float sh[];
#pragma unroll
    for (int k = 0; k < VEC; ++k) sh[threadIdx.x * VEC + k] = acc[k];
    __syncthreads();
    if (threadIdx.x < gpb && live) {
        float t[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) t[k] = 0.f;
        for (int q = threadIdx.x; q < static_cast<int>(blockDim.x); q += gpb)
#pragma unroll
            for (int k = 0; k < VEC; ++k) t[k] += sh[q * VEC + k];
#pragma unroll
        for (int k = 0; k < VEC; ++k) partial[static_cast<long long>(blockIdx.x) * u + g * VEC + k] = t[k];
    }
}

// bias[c] -= alpha * (sum_k partial[k][c]) * inv_b, one block per 32 columns:
// lane = column (coalesced rows of `partial`), threadIdx.y strides the chunks
// in ascending order, then a fixed-order sum over threadIdx.y (deterministic).
__global__ void __launch_bounds__(1024) bias_update_cols_kernel(const float* __restrict__ partial, int u, int chunks,
                                                                float* __restrict__ bias,
                                                                const double* __restrict__ alpha, float inv_b) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    __shared__ float sh[32][33];
    const int c = blockIdx.x * 32 + threadIdx.x;
    float s = 0.f;
    if (c < u) {
        // ascending k (fixed order), eight loads in flight per batch (the
        // plain loop compiled to one dependent L2 round trip per add)
        int k = threadIdx.y;
        for (; k + 7 * 32 < chunks; k += 8 * 32) {
            float t[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) t[i] = __ldg(partial + static_cast<long long>(k + 32 * i) * u + c);
#pragma unroll
            for (int i = 0; i < 8; ++i) s += t[i];
        }
        for (; k < chunks; k += 32) s += __ldg(partial + static_cast<long long>(k) * u + c);
    }
    sh[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.y == 0 && c < u) {
        float t = 0.f;
        for (int j = 0; j < 32; ++j) t += sh[j][threadIdx.x];
        bias[c] -= static_cast<float>(*alpha) * (t * inv_b);
    }
}

template <class T>
__global__ void convert_kernel(const T* __restrict__ src, int rows, int cols, float* __restrict__ dst,
                               long long ld) {
    const long long total = static_cast<long long>(rows) * cols;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / cols, c = i % cols;
        dst[r * ld + c] = static_cast<float>(src[i]);
    }
}

__global__ void finalize_kernel(StepState* st, const double* __restrict__ loss_row,
                                const int* __restrict__ correct_row, int b, double* loss_hist,
                                double* acc_hist, int hist_cap, int write_hist) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    double ls = 0.0;
    double cs = 0.0;
    if (write_hist) {
        // fixed-shape tree: thread i sums rows i, i+NT, ... in order
        for (int r = threadIdx.x; r < b; r += kRowThreads) {
            ls += loss_row[r];
            cs += correct_row[r];
        }
        ls = block_sum_d<kRowThreads>(ls);
        cs = block_sum_d<kRowThreads>(cs);
    }
    if (threadIdx.x == 0) {
        const int t = st->t;
        if (write_hist) {
            loss_hist[t % hist_cap] = ls / b;
            acc_hist[t % hist_cap] = cs / b;
        }
        if (st->diverge_flag && st->diverged_first == 0) st->diverged_first = t + 1;
        st->diverge_flag = 0;
        st->alpha *= 1.0 - st->decay;
        st->t = t + 1;
    }
}

template <class T>
__global__ void im2col_kernel(const T* __restrict__ src, int imgs, int H, int W, int C, int k, int p,
                              float* __restrict__ dst, long long ld) {
    const int Ho = H + 2 * p - k + 1, Wo = W + 2 * p - k + 1;
    const int kc = k * k * C;
    const long long total = static_cast<long long>(imgs) * Ho * Wo * kc;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int col = static_cast<int>(i % kc);
        const long long pix = i / kc;
        const int c = col % C, tap = col / C, r = tap / k, s = tap % k;
        const int wo = static_cast<int>(pix % Wo);
        const int ho = static_cast<int>((pix / Wo) % Ho);
        const long long n = pix / (static_cast<long long>(Wo) * Ho);
        const int hi = ho + r - p, wi = wo + s - p;
        float v = 0.f;
        if (hi >= 0 && hi < H && wi >= 0 && wi < W) v = static_cast<float>(src[((n * H + hi) * W + wi) * C + c]);
        dst[pix * ld + col] = v;
    }
}

// Generic conv path (grids the TMA boxes cannot tile, e.g. LeNet's 28x28 /
// 10x10): explicit im2col rows of a padded NHWC activation.  Column
// (tap, c) of output pixel (img, y, x) = x_pad[img][y + r][x + s][c] (the
// tensor's own zero ring is the conv padding); columns >= k*k*C are zero.
__global__ void im2col_act_kernel(const float* __restrict__ x, int imgs, int hp, int wp, long long ldx, int C, int k,
                                  int Ho, int Wo, float* __restrict__ dst, long long ldc, int st) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int kc = k * k * C;
    const long long total = static_cast<long long>(imgs) * Ho * Wo * ldc;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int col = static_cast<int>(i % ldc);
        const long long pix = i / ldc;
        float v = 0.f;
        if (col < kc) {
            const int c = col % C, tap = col / C, r = tap / k, s = tap % k;
            const int wo = static_cast<int>(pix % Wo);
            const int ho = static_cast<int>((pix / Wo) % Ho);
            const long long n = pix / (static_cast<long long>(Wo) * Ho);
            v = x[((n * hp + ho * st + r) * wp + wo * st + s) * ldx + c];
        }
        dst[i] = v;
    }
}

// Vectorised im2col for C % 4 == 0 (the generic path's strided convs, e.g.
// ResNet-18's stage transitions): thread = (output pixel, tap, 4 channels),
// one float4 load / store; consecutive threads walk a tap's contiguous
// channels, so reads and writes coalesce.  Columns >= k*k*C (row padding)
// are never written (zero since allocation).
template <class IDX>
__global__ void im2col_act_vec_kernel(const float* __restrict__ x, int imgs, int hp, int wp, long long ldx, int C,
                                      int k, int Ho, int Wo, float* __restrict__ dst, long long ldc, int st) {
    griddep_wait();
    const int groups = C >> 2, kk = k * k;
    const IDX total = static_cast<IDX>(imgs) * Ho * Wo * kk * groups;
    for (IDX i = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<IDX>(gridDim.x) * blockDim.x) {
        const int c4 = static_cast<int>(i % groups);
        const IDX t = i / groups;
        const int tap = static_cast<int>(t % kk);
        const IDX pix = t / kk;
        const int wo = static_cast<int>(pix % Wo);
        const IDX t2 = pix / Wo;
        const int ho = static_cast<int>(t2 % Ho);
        const long long n = static_cast<long long>(t2 / Ho);
        const int r = tap / k, s = tap - r * k;
        const float4 v = __ldg(reinterpret_cast<const float4*>(
            x + ((n * hp + ho * st + r) * wp + wo * st + s) * ldx + c4 * 4));
        *reinterpret_cast<float4*>(dst + static_cast<long long>(pix) * ldc + tap * C + c4 * 4) = v;
    }
}

// Vectorised col2im (C, c0, nc, ldk, ldo multiples of 4): thread = (input
// pixel, 4 channels of the destination slice); taps summed in ascending
// (r, s) order as col2im_kernel (same result bits).
template <class IDX>
__global__ void col2im_vec_kernel(const float* __restrict__ dcols, long long ldk, int imgs, int H, int W, int C, int k,
                                  int p, int Ho, int Wo, int c0, int nc, float* __restrict__ dst, long long ldo, int st) {
    griddep_wait();
    const int groups = nc >> 2;
    const IDX total = static_cast<IDX>(imgs) * H * W * groups;
    for (IDX i = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<IDX>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(i % groups);
        const IDX pix = i / groups;
        const int x = static_cast<int>(pix % W);
        const IDX t = pix / W;
        const int y = static_cast<int>(t % H);
        const long long n = static_cast<long long>(t / H);
        const int c = c0 + g * 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < k; ++r) {
            const int sy = y + p - r;
            if (sy < 0 || sy % st) continue;
            const int oy = sy / st;
            if (oy >= Ho) continue;
            for (int s = 0; s < k; ++s) {
                const int sx = x + p - s;
                if (sx < 0 || sx % st) continue;
                const int ox = sx / st;
                if (ox >= Wo) continue;
                const float4 v = __ldg(reinterpret_cast<const float4*>(
                    dcols + ((n * Ho + oy) * Wo + ox) * ldk + (r * k + s) * C + c));
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
        }
        *reinterpret_cast<float4*>(dst + static_cast<long long>(pix) * ldo + g * 4) = acc;
    }
}

// col2im_vec_kernel for k = 3: the nine taps unrolled, every valid tap's
// float4 load issued before the (ascending, same-bits) sum, so a thread has up
// to nine 16 B loads in flight instead of one (the runtime-k loop serialised
// them: 2.1 TB/s on ResNet-18's stride-2 transitions).
template <class IDX>
__global__ void col2im_k3_kernel(const float* __restrict__ dcols, long long ldk, int imgs, int H, int W, int C,
                                 int p, int Ho, int Wo, int c0, int nc, float* __restrict__ dst, long long ldo, int st) {
    griddep_wait();
    const int groups = nc >> 2;
    const IDX total = static_cast<IDX>(imgs) * H * W * groups;
    for (IDX i = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<IDX>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(i % groups);
        const IDX pix = i / groups;
        const int x = static_cast<int>(pix % W);
        const IDX t = pix / W;
        const int y = static_cast<int>(t % H);
        const long long n = static_cast<long long>(t / H);
        const int c = c0 + g * 4;
        int oy[3], ox[3];
        bool vy[3], vx[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int sy = y + p - r, sx = x + p - r;
            oy[r] = sy / st;
            ox[r] = sx / st;
            vy[r] = sy >= 0 && sy % st == 0 && oy[r] < Ho;
            vx[r] = sx >= 0 && sx % st == 0 && ox[r] < Wo;
        }
        float4 v[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                v[r * 3 + s] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (vy[r] && vx[s])
                    v[r * 3 + s] = __ldg(reinterpret_cast<const float4*>(
                        dcols + ((n * Ho + oy[r]) * Wo + ox[s]) * ldk + (r * 3 + s) * C + c));
            }
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s)
                if (vy[r] && vx[s]) {
                    acc.x += v[r * 3 + s].x;
                    acc.y += v[r * 3 + s].y;
                    acc.z += v[r * 3 + s].z;
                    acc.w += v[r * 3 + s].w;
                }
        *reinterpret_cast<float4*>(dst + static_cast<long long>(pix) * ldo + g * 4) = acc;
    }
}

// col2im for k = 3, stride 2 (ResNet's stage transitions): per dimension at
// most two taps reach an input position (t0 = (y + p) & 1 and t0 + 2), so a
// position sums <= 4 float4s; two positions per thread, every load of both
// issued before the sums (taps still added in ascending (r, s): same bits as
// col2im_kernel).
struct Col2imS2Taps {
    float4 v[4];
    bool ok[4];
};

__device__ __forceinline__ Col2imS2Taps col2im_s2_load(const float* __restrict__ dcols, long long ldk, int H, int W,
                                                       int C, int p, int Ho, int Wo, int c, long long n, int y,
                                                       int x) {
    const int ry = (y + p) & 1, rx = (x + p) & 1;
    int oy[2], ox[2], ty[2], tx[2];
    bool vy[2], vx[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        ty[q] = ry + 2 * q;
        tx[q] = rx + 2 * q;
        const int sy = y + p - ty[q], sx = x + p - tx[q];
        oy[q] = sy >> 1;
        ox[q] = sx >> 1;
        vy[q] = ty[q] < 3 && sy >= 0 && oy[q] < Ho;
        vx[q] = tx[q] < 3 && sx >= 0 && ox[q] < Wo;
    }
    Col2imS2Taps t;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int k = a * 2 + b;
            t.ok[k] = vy[a] && vx[b];
            t.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t.ok[k])
                t.v[k] = __ldg(reinterpret_cast<const float4*>(dcols + ((n * Ho + oy[a]) * Wo + ox[b]) * ldk +
                                                              (ty[a] * 3 + tx[b]) * C + c));
        }
    return t;
}

__device__ __forceinline__ float4 col2im_s2_sum(const Col2imS2Taps& t) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (t.ok[k]) {
            acc.x += t.v[k].x;
            acc.y += t.v[k].y;
            acc.z += t.v[k].z;
            acc.w += t.v[k].w;
        }
    return acc;
}

template <class IDX>
__global__ void col2im_k3s2_kernel(const float* __restrict__ dcols, long long ldk, int imgs, int H, int W, int C,
                                   int p, int Ho, int Wo, int c0, int nc, float* __restrict__ dst, long long ldo) {
    griddep_wait();
    const int groups = nc >> 2;
    const IDX total = static_cast<IDX>(imgs) * H * W * groups;
    const IDX stride = static_cast<IDX>(gridDim.x) * blockDim.x;
    for (IDX i = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; i < total; i += 2 * stride) {
        const IDX i2 = i + stride;
        const bool two = i2 < total;
        const int g = static_cast<int>(i % groups), g2 = two ? static_cast<int>(i2 % groups) : g;
        const IDX pix = i / groups, pix2 = two ? i2 / groups : pix;
        const int x = static_cast<int>(pix % W), x2 = static_cast<int>(pix2 % W);
        const IDX t = pix / W, t2 = pix2 / W;
        const int y = static_cast<int>(t % H), y2 = static_cast<int>(t2 % H);
        const long long n = static_cast<long long>(t / H), n2 = static_cast<long long>(t2 / H);
        const Col2imS2Taps a = col2im_s2_load(dcols, ldk, H, W, C, p, Ho, Wo, c0 + g * 4, n, y, x);
        Col2imS2Taps b;
        if (two) b = col2im_s2_load(dcols, ldk, H, W, C, p, Ho, Wo, c0 + g2 * 4, n2, y2, x2);
        *reinterpret_cast<float4*>(dst + static_cast<long long>(pix) * ldo + g * 4) = col2im_s2_sum(a);
        if (two) *reinterpret_cast<float4*>(dst + static_cast<long long>(pix2) * ldo + g2 * 4) = col2im_s2_sum(b);
    }
}

// col2im of the partial input gradient: g(img, y, x, c) for the input grid
// H x W = sum over taps (r, s) ascending of dcols[(img, y + p - r, x + p - s)]
// [(r*k + s)*C + c] over valid output positions (fixed order: deterministic).
// Channels [c0, c0 + nc) go to dst[(img*H + y)*W + x][c - c0] (a merge slot).
__global__ void col2im_kernel(const float* __restrict__ dcols, long long ldk, int imgs, int H, int W, int C, int k,
                              int p, int Ho, int Wo, int c0, int nc, float* __restrict__ dst, long long ldo, int st) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const long long total = static_cast<long long>(imgs) * H * W * nc;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int cc = static_cast<int>(i % nc);
        const long long pix = i / nc;
        const int x = static_cast<int>(pix % W);
        const int y = static_cast<int>((pix / W) % H);
        const long long n = pix / (static_cast<long long>(W) * H);
        const int c = c0 + cc;
        float g = 0.f;
        for (int r = 0; r < k; ++r) {
            const int sy = y + p - r;  // = oy * st
            if (sy < 0 || sy % st) continue;
            const int oy = sy / st;
            if (oy >= Ho) continue;
            for (int s = 0; s < k; ++s) {
                const int sx = x + p - s;
                if (sx < 0 || sx % st) continue;
                const int ox = sx / st;
                if (ox >= Wo) continue;
                g += dcols[((n * Ho + oy) * Wo + ox) * ldk + (r * k + s) * C + c];
            }
        }
        dst[pix * ldo + cc] = g;
    }
}

// Small-grid conv as a dense layer ("dense conv", e.g. VGG's 2x2 layers):
// with P = Ho*Wo output and Q = H*W input positions, the conv is
//   out[n][(p, co)] = sum_{(q, ci)} in[n][(q, ci)] * Wx[(p, co)][(q, ci)]
//   Wx[(p, co)][(q, ci)] = W[co][tap(p, q)][ci],  tap = (qy - py + pad, qx - px + pad)
// (zero when the tap falls outside the kernel).  W stays the parameter
// ([u][k*k][ck], the implicit-GEMM layout); Wx is re-expanded after every
// update.  The wgrad GEMM yields dWx; the fold sums dWx over the (p, q) pairs
// of each tap in ascending (p, q) order (deterministic), applies SGD to W and
// rewrites Wx.  Thread = one (co, ci) pair.
__device__ __forceinline__ int dc_tap(const DenseConvGeom& g, int p, int q) {
    const int py = p / g.Wo, px = p - py * g.Wo, qy = q / g.W, qx = q - qy * g.W;
    const int r = qy - py + g.pad, s = qx - px + g.pad;
    return (r >= 0 && r < g.k && s >= 0 && s < g.k) ? r * g.k + s : -1;
}

__global__ void dense_conv_expand_kernel(DenseConvGeom g, const float* __restrict__ W, float* __restrict__ Wx) {
    const int P = g.Ho * g.Wo, Q = g.H * g.W;
    const long long total = static_cast<long long>(g.u) * g.C;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int co = static_cast<int>(i / g.C), ci = static_cast<int>(i % g.C);
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q) {
                const int t = dc_tap(g, p, q);
                Wx[static_cast<long long>(p * g.u + co) * g.ldx + q * g.C + ci] =
                    t >= 0 ? W[co * g.ldw + t * g.ck + ci] : 0.f;
            }
    }
}

// 3x3 / pad 1 on a 2x2 grid (VGG conv11-13), fully unrolled: 16 (p, q)
// pairs onto 9 taps, summed in ascending (p, q) order.  Extra blocks past the
// (co, ci) range apply the bias update from the merge's partial rows (lane =
// column, 8 phases over the chunks, fixed-order sum).
__global__ void __launch_bounds__(256) dense_conv_update_2x2_kernel(
    DenseConvGeom g, const float* __restrict__ dWx, float* __restrict__ W, float* __restrict__ Wx,
    const double* __restrict__ alpha, float inv_b, int* flag, const float* __restrict__ bpart, int bchunks,
    float* __restrict__ bias) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const float a = static_cast<float>(*alpha);
    const long long total = static_cast<long long>(g.u) * g.C;
    // bias blocks first (they start with the grid): warp = column, lane =
    // phase over the chunks (k = lane, lane + 32, ...), fixed butterfly
    const int bblocks = bias != nullptr ? (g.u + 7) / 8 : 0;
    if (static_cast<int>(blockIdx.x) < bblocks) {
        const int col = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
        float acc = 0.f;
        if (col < g.u) {
#pragma unroll 8
            for (int k = lane; k < bchunks; k += 32) acc += bpart[static_cast<long long>(k) * g.u + col];
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0 && col < g.u) bias[col] -= a * (acc * inv_b);
        return;
    }
    const long long i = (blockIdx.x - bblocks) * 256LL + threadIdx.x;
    if (i >= total) return;
    dense_conv_update_2x2_item(g, dWx, W, Wx, a, inv_b, flag, i);
}

__global__ void dense_conv_fold_sgd_kernel(DenseConvGeom g, const float* __restrict__ dWx, float* __restrict__ W,
                                           float* __restrict__ Wx, const double* __restrict__ alpha, float inv_b,
                                           int* flag) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int P = g.Ho * g.Wo, Q = g.H * g.W;
    const float a = static_cast<float>(*alpha);
    const long long total = static_cast<long long>(g.u) * g.C;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int co = static_cast<int>(i / g.C), ci = static_cast<int>(i % g.C);
        float gsum[25];
#pragma unroll
        for (int t = 0; t < 25; ++t) gsum[t] = 0.f;
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q) {
                const int t = dc_tap(g, p, q);
                if (t < 0) continue;
                const float v = dWx[static_cast<long long>(p * g.u + co) * g.ldx + q * g.C + ci];
#pragma unroll
                for (int tt = 0; tt < 25; ++tt)
                    if (tt == t) gsum[tt] += v;
            }
        bool bad = false;
        float wn[25];
#pragma unroll
        for (int t = 0; t < 25; ++t) {
            wn[t] = 0.f;
            if (t < g.k * g.k) {
                const float gr = gsum[t] * inv_b;
                bad |= !isfinite(gr);
                float* w = W + co * g.ldw + t * g.ck + ci;
                wn[t] = *w - a * gr;
                *w = wn[t];
            }
        }
        if (bad && flag != nullptr) atomicOr(flag, 1);
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < Q; ++q) {
                const int t = dc_tap(g, p, q);
                float v = 0.f;
#pragma unroll
                for (int tt = 0; tt < 25; ++tt)
                    if (tt == t) v = wn[tt];
                Wx[static_cast<long long>(p * g.u + co) * g.ldx + q * g.C + ci] = v;
            }
    }
}

// im2col of the fp32 input for K = k*k*C <= 32 (VGG conv1 27, LeNet C1 25):
// 8 threads per output pixel, thread g writes columns 4g .. 4g+3 of the
// pixel's 32-column row (zeros past K) as one float4, so a warp stores four
// whole 128 B rows (coalesced); the gathered reads hit L1 / L2 (the input is
// a few MB).
template <class T>
__global__ void __launch_bounds__(256) im2col_row32_kernel(const T* __restrict__ src, int imgs, int H, int W,
                                                           int C, int k, int p, float* __restrict__ dst,
                                                           long long ld) {
    // blockIdx.y = image, 8 threads per output pixel (one float4 of the
    // 32-float row each).  The column -> (row tap, column tap, channel) map is
    // a 32-entry shared table built once per block: the per-element integer
    // divisions by the runtime C and k made this kernel instruction-bound
    // (60 us for 67 MB of rows).
    __shared__ int tap_off[32];  // (dh * W + dw) * C + c relative to (ho - p, wo - p); -1: padding column
    __shared__ short tap_dh[32], tap_dw[32];
    const int K = k * k * C;
    if (threadIdx.x < 32) {
        const int col = threadIdx.x;
        if (col < K) {
            const int tap = col / C, c = col - tap * C;
            const int rr = tap / k, ss = tap - rr * k;
            tap_off[col] = (rr * W + ss) * C + c;
            tap_dh[col] = static_cast<short>(rr);
            tap_dw[col] = static_cast<short>(ss);
        } else {
            tap_off[col] = -1;
        }
    }
    __syncthreads();
    const int Ho = H + 2 * p - k + 1, Wo = W + 2 * p - k + 1;
    const int n = blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int pi = t >> 3, g = t & 7;
    if (pi >= Ho * Wo) return;
    const int ho = pi / Wo, wo = pi - ho * Wo;
    const T* img = src + static_cast<long long>(n) * H * W * C;
    const int base = ((ho - p) * W + (wo - p)) * C;  // may be negative; only in-image taps are read
    float r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int col = 4 * g + e;
        const int off = tap_off[col];
        const int hi = ho - p + tap_dh[col], wi = wo - p + tap_dw[col];
        r[e] = (off >= 0 && hi >= 0 && hi < H && wi >= 0 && wi < W) ? static_cast<float>(__ldg(img + base + off)) : 0.f;
    }
    reinterpret_cast<float4*>(dst + (static_cast<long long>(n) * Ho * Wo + pi) * ld)[g] =
        make_float4(r[0], r[1], r[2], r[3]);
}

template <class T>
__global__ void pad_input_kernel(const T* __restrict__ src, int imgs, int H, int W, int C, float* __restrict__ dst,
                                 int p, long long ld) {
    const long long total = static_cast<long long>(imgs) * H * W * C;
    const int hp = H + 2 * p, wp = W + 2 * p;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % C);
        long long pix = i / C;
        const int w = static_cast<int>(pix % W);
        pix /= W;
        const int h = static_cast<int>(pix % H);
        const long long n = pix / H;
        dst[((n * hp + h + p) * wp + w + p) * ld + c] = static_cast<float>(src[i]);
    }
}

// Threads own a fixed group of VEC channels for the whole grid-stride loop
// (blockDim and the grid stride are multiples of the group count), which keeps
// loads/stores vectorised along channels and lets conv_merge accumulate the
// bias gradient of its channels in registers.
template <int VEC, class IDX>
__global__ void pool_fwd_kernel(const float* __restrict__ U, long long ldu, int imgs, int Ho, int Wo, int uch,
                                int pool, unsigned char* __restrict__ argmax, ActLayout out, PoolDsts dsts) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int Hq = Ho / pool, Wq = Wo / pool;
    const IDX groups = uch / VEC;
    const IDX total = static_cast<IDX>(imgs) * Hq * Wq * groups;
    for (IDX i = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<IDX>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(i % groups);
        const IDX pp = i / groups;  // pooled pixel
        const int x = static_cast<int>(pp % Wq);
        const IDX t = pp / Wq;
        const int y = static_cast<int>(t % Hq);
        const long long n = t / Hq;
        const int c0 = g * VEC;
        float v[VEC];
        unsigned char arg[VEC];
        if (pool == 1) {
            if (VEC == 4) {
                const float4 a = *reinterpret_cast<const float4*>(U + static_cast<long long>(pp) * ldu + c0);
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            } else {
                v[0] = U[static_cast<long long>(pp) * ldu + c0];
            }
        } else {
            const long long base = (n * Ho + 2 * y) * Wo + 2 * x;
            const long long offs[4] = {base, base + 1, base + Wo, base + Wo + 1};
            static_assert(sizeof(IDX) >= 4, "index type");
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                v[k] = -INFINITY;
                arg[k] = 0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float e[VEC];
                if (VEC == 4) {
                    const float4 a = *reinterpret_cast<const float4*>(U + offs[q] * ldu + c0);
                    e[0] = a.x; e[1] = a.y; e[2] = a.z; e[3] = a.w;
                } else {
                    e[0] = U[offs[q] * ldu + c0];
                }
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (q == 0 || e[k] > v[k]) {  // first max wins
                        v[k] = e[k];
                        arg[k] = static_cast<unsigned char>(q);
                    }
            }
#pragma unroll
            for (int k = 0; k < VEC; ++k) argmax[static_cast<long long>(pp) * uch + c0 + k] = arg[k];
        }
        if (out.kind == 0) {
            const long long o = ((n * out.hp + y + out.pad) * out.wp + x + out.pad) * out.ld + out.col0 + c0;
            for (int d = 0; d < dsts.n; ++d) {
                if (VEC == 4) *reinterpret_cast<float4*>(dsts.ptr[d] + o) = make_float4(v[0], v[1], v[2], v[3]);
                else dsts.ptr[d][o] = v[0];
            }
        } else {
            for (int k = 0; k < VEC; ++k) {
                const long long o = n * out.ld + static_cast<long long>(out.col0 + c0 + k) * Hq * Wq +
                                    static_cast<long long>(y) * Wq + x;
                for (int d = 0; d < dsts.n; ++d) dsts.ptr[d][o] = v[k];
            }
        }
    }
}

template <int VEC, class IDX>
__global__ void conv_merge_kernel(ConvMerge m, float* __restrict__ db_partial) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int groups = m.uch / VEC;
    const IDX total = static_cast<IDX>(m.imgs) * m.Ho * m.Wo * groups;
    const int Hg = m.Ho / m.pool, Wg = m.Wo / m.pool;
    const int hq = m.Ho + 2 * m.q, wq = m.Wo + 2 * m.q;
    float db[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) db[k] = 0.f;
    const IDX start = blockIdx.x * static_cast<IDX>(blockDim.x) + threadIdx.x;
    const int g = static_cast<int>(start % groups);  // constant: blockDim and the stride are multiples of groups
    const int c0 = g * VEC;
    for (IDX i = start; i < total; i += static_cast<IDX>(gridDim.x) * blockDim.x) {
        const IDX pix = i / groups;
        const int w = static_cast<int>(pix % m.Wo);
        const IDX t = pix / m.Wo;
        const int h = static_cast<int>(t % m.Ho);
        const long long n = t / m.Ho;
        float gr[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) gr[k] = 0.f;
        int y = h, x = w;
        bool in_grid = true;
        if (m.pool == 2) {
            y = h >> 1;
            x = w >> 1;
            in_grid = y < Hg && x < Wg;
        }
        if (in_grid) {
            const long long gp = (n * Hg + y) * Wg + x;
            if (m.slot_kind == 0) {
                const long long idx = gp * m.lds + c0;
                for (int s = 0; s < m.slots.n; ++s) {
                    if (VEC == 4) {
                        const float4 a = *reinterpret_cast<const float4*>(m.slots.slot[s] + idx);
                        gr[0] += a.x; gr[1] += a.y; gr[2] += a.z; gr[3] += a.w;
                    } else {
                        gr[0] += m.slots.slot[s][idx];
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < VEC; ++k) {
                    const long long idx = n * m.lds + static_cast<long long>(c0 + k) * Hg * Wg + y * Wg + x;
                    for (int s = 0; s < m.slots.n; ++s) gr[k] += m.slots.slot[s][idx];
                }
            }
            if (m.pool == 2) {
                const unsigned char want = static_cast<unsigned char>(((h & 1) << 1) | (w & 1));
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (m.argmax[gp * m.uch + c0 + k] != want) gr[k] = 0.f;
            }
        }
        if (m.mask_kind == 1) {
            const float* up = m.U + static_cast<long long>(pix) * m.ldu + c0;
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (!(up[k] > 0.f)) gr[k] = 0.f;
        } else if (m.mask_kind == 2) {
            const ActLayout& a = m.act_layout;
            const float* ap = m.act + ((n * a.hp + h + a.pad) * a.wp + w + a.pad) * a.ld + a.col0 + c0;
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (!(ap[k] > 0.f)) gr[k] = 0.f;
        } else if (m.mask_kind == 3 && (h >> 1) < m.Ho / 2 && (w >> 1) < m.Wo / 2) {
            // pooled activation at the window: the max = U at the argmax, the only
            // position the routing above leaves non-zero
            const ActLayout& a = m.act_layout;
            const float* ap = m.act + ((n * a.hp + (h >> 1) + a.pad) * a.wp + (w >> 1) + a.pad) * a.ld + a.col0 + c0;
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                if (!(ap[k] > 0.f)) gr[k] = 0.f;
        }
        float* out = m.d_pad + ((n * hq + h + m.q) * wq + w + m.q) * m.ldd + c0;
        if (VEC == 4) {
            *reinterpret_cast<float4*>(out) = make_float4(gr[0], gr[1], gr[2], gr[3]);
        } else {
            out[0] = gr[0];
        }
#pragma unroll
        for (int k = 0; k < VEC; ++k) db[k] += gr[k];
    }
    // deterministic per-block channel partials: threads of the same channel
    // group are threadIdx.x = g' + groups * j; sum them in j order
    extern __shared__ float sh[];
#pragma unroll
    for (int k = 0; k < VEC; ++k) sh[threadIdx.x * VEC + k] = db[k];
    __syncthreads();
    if (threadIdx.x < groups) {
        float acc[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc[k] = 0.f;
        for (int t = threadIdx.x; t < static_cast<int>(blockDim.x); t += groups)
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc[k] += sh[t * VEC + k];
#pragma unroll
        for (int k = 0; k < VEC; ++k)
            db_partial[static_cast<long long>(blockIdx.x) * m.uch + threadIdx.x * VEC + k] = acc[k];
    }
}

// Vectorised conv_merge (slot_kind 0, VEC 4): one image row (n, h) per block
// iteration, thread = (pixel column w, channel group g) with g fixed for the
// thread.  Index math is per row; the U pixels a thread owns in a row are
// loaded first (slot, argmax, mask) and then combined, so each thread keeps
// ~3U independent loads in flight instead of a dependent chain per element.
template <int U>
__global__ void conv_merge_rows_kernel(ConvMerge m, float* __restrict__ db_partial) {
    griddep_wait();  // programmatic launch: the predecessor's results are visible after this
    const int groups = m.uch >> 2;
    const int g = threadIdx.x % groups;
    const int c0 = g * 4;
    const int wstep = blockDim.x / groups;
    const int w0 = threadIdx.x / groups;
    const int Hg = m.Ho / m.pool, Wg = m.Wo / m.pool;
    const int hq = m.Ho + 2 * m.q, wq = m.Wo + 2 * m.q;
    const int rows = m.imgs * m.Ho;
    const ActLayout& a = m.act_layout;
    float4 db = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* s0 = m.slots.n > 0 ? m.slots.slot[0] : nullptr;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const int n = r / m.Ho, h = r - n * m.Ho;
        const int y = m.pool == 2 ? h >> 1 : h;
        const bool row_in = y < Hg;
        const long long grow = (static_cast<long long>(n) * Hg + y) * Wg;
        const float* arow = m.mask_kind == 2
                                ? m.act + ((static_cast<long long>(n) * a.hp + h + a.pad) * a.wp + a.pad) * a.ld + a.col0 + c0
                            : m.mask_kind == 3 && row_in
                                ? m.act + ((static_cast<long long>(n) * a.hp + y + a.pad) * a.wp + a.pad) * a.ld + a.col0 + c0
                                : nullptr;
        const float* urow = m.mask_kind == 1 ? m.U + static_cast<long long>(r) * m.Wo * m.ldu + c0 : nullptr;
        float* orow = m.d_pad + ((static_cast<long long>(n) * hq + h + m.q) * wq + m.q) * m.ldd + c0;
        for (int wb = w0; wb < m.Wo; wb += U * wstep) {
            float4 gr[U];
            uint32_t am[U];
            float4 mk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int w = wb + u * wstep;
                gr[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                am[u] = 0;
                mk[u] = make_float4(1.f, 1.f, 1.f, 1.f);
                if (w >= m.Wo) continue;
                const int x = m.pool == 2 ? w >> 1 : w;
                // first slot, argmax and mask issued before the extra slots' loop
                // (the loop between them serialised the position's round trips)
                float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f);
                const bool in = row_in && x < Wg;
                const long long gp = grow + x;
                if (in) {
                    if (s0 != nullptr) t0 = __ldg(reinterpret_cast<const float4*>(s0 + gp * m.lds + c0));
                    if (m.pool == 2) am[u] = __ldg(reinterpret_cast<const uint32_t*>(m.argmax + gp * m.uch + c0));
                } else {
                    am[u] = 0xffffffffu;  // outside the pooled grid: no gradient
                }
                if (m.mask_kind == 2) mk[u] = __ldg(reinterpret_cast<const float4*>(arow + static_cast<long long>(w) * a.ld));
                else if (m.mask_kind == 3 && in)
                    mk[u] = __ldg(reinterpret_cast<const float4*>(arow + static_cast<long long>(x) * a.ld));
                else if (m.mask_kind == 1) mk[u] = __ldg(reinterpret_cast<const float4*>(urow + static_cast<long long>(w) * m.ldu));
                if (in) {
                    gr[u].x += t0.x; gr[u].y += t0.y; gr[u].z += t0.z; gr[u].w += t0.w;
                    for (int s = 1; s < m.slots.n; ++s) {
                        const float4 v = __ldg(reinterpret_cast<const float4*>(m.slots.slot[s] + gp * m.lds + c0));
                        gr[u].x += v.x; gr[u].y += v.y; gr[u].z += v.z; gr[u].w += v.w;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int w = wb + u * wstep;
                if (w >= m.Wo) continue;
                float4 v = gr[u];
                if (m.pool == 2) {  // outside the pooled grid gr is 0 already
                    const uint32_t want = static_cast<uint32_t>(((h & 1) << 1) | (w & 1));
                    const uint32_t b = am[u];
                    if ((b & 0xffu) != want) v.x = 0.f;
                    if (((b >> 8) & 0xffu) != want) v.y = 0.f;
                    if (((b >> 16) & 0xffu) != want) v.z = 0.f;
                    if ((b >> 24) != want) v.w = 0.f;
                }
                if (!(mk[u].x > 0.f)) v.x = 0.f;
                if (!(mk[u].y > 0.f)) v.y = 0.f;
                if (!(mk[u].z > 0.f)) v.z = 0.f;
                if (!(mk[u].w > 0.f)) v.w = 0.f;
                *reinterpret_cast<float4*>(orow + static_cast<long long>(w) * m.ldd) = v;
                db.x += v.x; db.y += v.y; db.z += v.z; db.w += v.w;
            }
        }
    }
    extern __shared__ float sh[];
    reinterpret_cast<float4*>(sh)[threadIdx.x] = db;
    __syncthreads();
    if (threadIdx.x < groups) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = threadIdx.x; t < static_cast<int>(blockDim.x); t += groups) {
            const float4 v = reinterpret_cast<const float4*>(sh)[t];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        *reinterpret_cast<float4*>(db_partial + static_cast<long long>(blockIdx.x) * m.uch + c0) = acc;
    }
}


__global__ void unpack_gather_kernel(const float* __restrict__ recv, int g, int rows, int u, float* __restrict__ dst,
                                     long long ld) {
    const long long total = static_cast<long long>(g) * rows * u;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % u);
        const long long t = i / u;
        const int r = static_cast<int>(t % rows);
        const int k = static_cast<int>(t / rows);
        dst[static_cast<long long>(r) * ld + static_cast<long long>(k) * u + c] = recv[i];
    }
}

// ---------------------------------------------------------------- residual extension

// Thread = (image, pooled pixel, 4-channel group); window p x p (p = 1: no
// pooling).  Deterministic: the window is summed in row-major order.
__global__ void residual_act_kernel(float* __restrict__ U, long long ldu, int imgs, int Ho, int Wo, int uch, int c0,
                                    int relu, int pool, SkipSrc skip, ActLayout out, PoolDsts dsts, int write_u,
                                    int skip_vec) {
    griddep_wait();
    const int Hq = Ho / pool, Wq = Wo / pool;
    const int groups = uch >> 2;
    const long long total = static_cast<long long>(imgs) * Hq * Wq * groups;
    const float inv = 1.f / static_cast<float>(pool * pool);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(i % groups);
        const long long pp = i / groups;
        const int x = static_cast<int>(pp % Wq);
        const long long t = pp / Wq;
        const int y = static_cast<int>(t % Hq);
        const long long n = t / Hq;
        const int c = g * 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int dy = 0; dy < pool; ++dy) {
            for (int dx = 0; dx < pool; ++dx) {
                const int h = y * pool + dy, w = x * pool + dx;
                float4* up = reinterpret_cast<float4*>(U + ((n * Ho + h) * Wo + w) * ldu + c);
                float4 u = *up;
                if (skip.a != nullptr) {  // option A: position (f h, f w) of the source
                    const long long sb = ((n * skip.lay.hp + h * skip.f + skip.lay.pad) * skip.lay.wp + w * skip.f +
                                          skip.lay.pad) * skip.lay.ld;
                    const int ca = c0 + c;  // absolute channel of lane k: ca + k
                    if (skip_vec && ca + 4 <= skip.C) {  // whole 4-channel group inside C_s: one 16 B load
                        const float4 sv = __ldg(reinterpret_cast<const float4*>(skip.a + sb + ca));
                        u.x += sv.x; u.y += sv.y; u.z += sv.z; u.w += sv.w;
                    } else {
                        if (ca + 0 < skip.C) u.x += __ldg(skip.a + sb + ca + 0);
                        if (ca + 1 < skip.C) u.y += __ldg(skip.a + sb + ca + 1);
                        if (ca + 2 < skip.C) u.z += __ldg(skip.a + sb + ca + 2);
                        if (ca + 3 < skip.C) u.w += __ldg(skip.a + sb + ca + 3);
                    }
                    // the pre-activation is kept only where the backward mask needs it
                    // (pooled output); otherwise the mask reads the activation itself
                    if (write_u) *up = u;
                }
                if (relu) {
                    u.x = u.x > 0.f ? u.x : 0.f;
                    u.y = u.y > 0.f ? u.y : 0.f;
                    u.z = u.z > 0.f ? u.z : 0.f;
                    u.w = u.w > 0.f ? u.w : 0.f;
                }
                acc.x += u.x;
                acc.y += u.y;
                acc.z += u.z;
                acc.w += u.w;
            }
        }
        if (pool > 1) {
            acc.x *= inv;
            acc.y *= inv;
            acc.z *= inv;
            acc.w *= inv;
        }
        if (out.kind == 0) {
            const long long o = ((n * out.hp + y + out.pad) * out.wp + x + out.pad) * out.ld + out.col0 + c;
            for (int d = 0; d < dsts.n; ++d) *reinterpret_cast<float4*>(dsts.ptr[d] + o) = acc;
        } else {
            const float v[4] = {acc.x, acc.y, acc.z, acc.w};
            for (int k = 0; k < 4; ++k) {
                const long long o = n * out.ld + static_cast<long long>(out.col0 + c + k) * Hq * Wq +
                                    static_cast<long long>(y) * Wq + x;
                for (int d = 0; d < dsts.n; ++d) dsts.ptr[d][o] = v[k];
            }
        }
    }
}

// conv_merge_rows_kernel's structure (block = image row, threads = (column,
// 4-channel group), bias partial per block in fixed order) with average-pool
// routing and the shortcut term.
// 592 blocks = 4 per SM: the register cap keeps all four resident (a fifth
// wave of 3-per-SM residency measured +40 % on the 32x32 layers)
template <bool COL2IM>
__global__ void __launch_bounds__(256, 4)
conv_merge_res_kernel(ConvMerge m, int pool_avg, SkipGrad sg, Col2imSrc cx, float* __restrict__ db_partial) {
    griddep_wait();
    const int groups = m.uch >> 2;
    const int g = threadIdx.x % groups;
    const int c0 = g * 4;
    const int wstep = blockDim.x / groups;
    const int w0 = threadIdx.x / groups;
    const int p = m.pool;
    const int Hg = m.Ho / p, Wg = m.Wo / p;
    const int hq = m.Ho + 2 * m.q, wq = m.Wo + 2 * m.q;
    const int rows = m.imgs * m.Ho;
    const ActLayout& a = m.act_layout;
    const float inv = 1.f / static_cast<float>(p * p);
    float4 db = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* s0 = m.slots.n > 0 ? m.slots.slot[0] : nullptr;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
        const int n = r / m.Ho, h = r - n * m.Ho;
        const int y = h / p;
        for (int w = w0; w < m.Wo; w += wstep) {
            const int x = w / p;
            const long long gp = (static_cast<long long>(n) * Hg + y) * Wg + x;
            // every load of the position issued before the first use (one
            // round trip instead of three dependent ones)
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            float4 t0 = zero;
            Col2imS2Taps ct;
            if (COL2IM)
                ct = col2im_s2_load(cx.dcols, cx.ldk, m.Ho, m.Wo, cx.C, cx.p, cx.Ho, cx.Wo, cx.c0 + c0, n, h, w);
            else if (s0 != nullptr)
                t0 = __ldg(reinterpret_cast<const float4*>(s0 + gp * m.lds + c0));
            const bool amax = p == 2 && !pool_avg;
            const uint32_t b = amax ? __ldg(reinterpret_cast<const uint32_t*>(m.argmax + gp * m.uch + c0)) : 0u;
            const bool has_sg = sg.d != nullptr && h % sg.f == 0 && w % sg.f == 0;
            const float4 ts = has_sg ? __ldg(reinterpret_cast<const float4*>(
                                           sg.d + ((static_cast<long long>(n) * sg.hq + h / sg.f + sg.q) * sg.wq +
                                                   w / sg.f + sg.q) * sg.ldd + sg.c0 + c0))
                                     : zero;
            float4 mk = make_float4(1.f, 1.f, 1.f, 1.f);
            if (m.mask_kind == 1)
                mk = __ldg(reinterpret_cast<const float4*>(m.U + (static_cast<long long>(r) * m.Wo + w) * m.ldu + c0));
            else if (m.mask_kind == 2)
                mk = __ldg(reinterpret_cast<const float4*>(
                    m.act + ((static_cast<long long>(n) * a.hp + h + a.pad) * a.wp + w + a.pad) * a.ld + a.col0 + c0));
            if (COL2IM) t0 = col2im_s2_sum(ct);
            float4 v = zero;
            v.x += t0.x; v.y += t0.y; v.z += t0.z; v.w += t0.w;
            for (int s = 1; s < m.slots.n; ++s) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(m.slots.slot[s] + gp * m.lds + c0));
                v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w;
            }
            if (amax) {  // max pool: the argmax position of the window takes it
                const uint32_t want = static_cast<uint32_t>(((h & 1) << 1) | (w & 1));
                if ((b & 0xffu) != want) v.x = 0.f;
                if (((b >> 8) & 0xffu) != want) v.y = 0.f;
                if (((b >> 16) & 0xffu) != want) v.z = 0.f;
                if ((b >> 24) != want) v.w = 0.f;
            } else if (p > 1) {
                v.x *= inv; v.y *= inv; v.z *= inv; v.w *= inv;
            }
            if (has_sg) {
                v.x += ts.x; v.y += ts.y; v.z += ts.z; v.w += ts.w;
            }
            if (!(mk.x > 0.f)) v.x = 0.f;
            if (!(mk.y > 0.f)) v.y = 0.f;
            if (!(mk.z > 0.f)) v.z = 0.f;
            if (!(mk.w > 0.f)) v.w = 0.f;
            *reinterpret_cast<float4*>(m.d_pad + ((static_cast<long long>(n) * hq + h + m.q) * wq + w + m.q) * m.ldd +
                                       c0) = v;
            db.x += v.x; db.y += v.y; db.z += v.z; db.w += v.w;
        }
    }
    extern __shared__ float sh[];
    reinterpret_cast<float4*>(sh)[threadIdx.x] = db;
    __syncthreads();
    if (threadIdx.x < groups) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = threadIdx.x; t < static_cast<int>(blockDim.x); t += groups) {
            const float4 u = reinterpret_cast<const float4*>(sh)[t];
            acc.x += u.x; acc.y += u.y; acc.z += u.z; acc.w += u.w;
        }
        *reinterpret_cast<float4*>(db_partial + static_cast<long long>(blockIdx.x) * m.uch + c0) = acc;
    }
}

int grid_for(long long work, int threads) {
    long long g = (work + threads - 1) / threads;
    const long long cap = 148LL * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_loss_head(const float* in, long long ld_in, int rows, int F, const int* labels,
                             int loss_kind, int relu_last, const LossTargets& t, double* loss_row,
                             int* correct_row, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    pdl_launch(loss_head_kernel, dim3(rows), dim3(kRowThreads), 0, s, in, ld_in, F, labels, loss_kind, relu_last, t,
                                                  loss_row, correct_row);
    return cudaGetLastError();
}

cudaError_t launch_reduce_mask(const ReduceSlots& slots, long long ld_slot, int rows, int cols,
                               const float* mask, long long ld_mask, float* out, long long ld_out,
                               cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    bool vec = (cols % 4 == 0) && (ld_slot % 4 == 0) && (ld_out % 4 == 0) &&
               (mask == nullptr || ld_mask % 4 == 0) &&
               (reinterpret_cast<uintptr_t>(out) % 16 == 0) &&
               (mask == nullptr || reinterpret_cast<uintptr_t>(mask) % 16 == 0);
    for (int k = 0; k < slots.n; ++k) vec = vec && reinterpret_cast<uintptr_t>(slots.slot[k]) % 16 == 0;
    const long long work = static_cast<long long>(rows) * (vec ? cols / 4 : cols);
    pdl_launch(reduce_mask_kernel, dim3(grid_for(work, 256)), dim3(256), 0, s, slots, ld_slot, rows, cols, mask, ld_mask,
                                                           out, ld_out, vec);
    return cudaGetLastError();
}

cudaError_t launch_bias_update(const float* delta, long long ld, long long rows, int u, float* partial,
                               float* bias, const double* alpha, float inv_b, cudaStream_t s) {
    if (u <= 0) return cudaSuccess;
    const int chunks = colsum_chunks(rows);
    const bool v4 = u % 4 == 0 && ld % 4 == 0 && reinterpret_cast<uintptr_t>(delta) % 16 == 0;
    const int groups = v4 ? u / 4 : u;
    const int gpb = groups < 256 ? groups : 256;
    const int block = (256 / gpb) * gpb;
    const dim3 grid(chunks, (groups + gpb - 1) / gpb);
    const size_t shmem = sizeof(float) * block * (v4 ? 4 : 1);
    if (v4) pdl_launch(colsum_rows_kernel<4>, dim3(grid), dim3(block), shmem, s, delta, ld, rows, u, partial);
    else pdl_launch(colsum_rows_kernel<1>, dim3(grid), dim3(block), shmem, s, delta, ld, rows, u, partial);
    pdl_launch(bias_update_cols_kernel, dim3((u + 31) / 32), dim3(dim3(32, 32)), 0, s, partial, u, chunks, bias, alpha, inv_b);
    return cudaGetLastError();
}

cudaError_t launch_colsum(const float* delta, long long ld, long long rows, int u, float* partial, cudaStream_t s) {
    if (u <= 0 || rows <= 0) return cudaSuccess;
    const int chunks = colsum_chunks(rows);
    const bool v4 = u % 4 == 0 && ld % 4 == 0 && reinterpret_cast<uintptr_t>(delta) % 16 == 0;
    const int groups = v4 ? u / 4 : u;
    const int gpb = groups < 256 ? groups : 256;
    const int block = (256 / gpb) * gpb;
    const dim3 grid(chunks, (groups + gpb - 1) / gpb);
    const size_t shmem = sizeof(float) * block * (v4 ? 4 : 1);
    if (v4) pdl_launch(colsum_rows_kernel<4>, dim3(grid), dim3(block), shmem, s, delta, ld, rows, u, partial);
    else pdl_launch(colsum_rows_kernel<1>, dim3(grid), dim3(block), shmem, s, delta, ld, rows, u, partial);
    return cudaGetLastError();
}

cudaError_t launch_convert_f64(const double* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s) {
    const long long n = static_cast<long long>(rows) * cols;
    if (n <= 0) return cudaSuccess;
    convert_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(src, rows, cols, dst, ld);
    return cudaGetLastError();
}

cudaError_t launch_convert_f32(const float* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s) {
    const long long n = static_cast<long long>(rows) * cols;
    if (n <= 0) return cudaSuccess;
    convert_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(src, rows, cols, dst, ld);
    return cudaGetLastError();
}

cudaError_t launch_im2col_input(const double* src64, const float* src32, int imgs, int H, int W, int C, int k,
                                int p, float* dst, long long ld, cudaStream_t s) {
    const long long n = static_cast<long long>(imgs) * (H + 2 * p - k + 1) * (W + 2 * p - k + 1) * k * k * C;
    if (n <= 0) return cudaSuccess;
    const long long npix = n / (static_cast<long long>(k) * k * C);
    if (k * k * C <= 32 && ld == 32 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        const dim3 blocks(static_cast<unsigned>((npix / imgs * 8 + 255) / 256), static_cast<unsigned>(imgs));
        if (src32 != nullptr) im2col_row32_kernel<float><<<blocks, 256, 0, s>>>(src32, imgs, H, W, C, k, p, dst, ld);
        else im2col_row32_kernel<double><<<blocks, 256, 0, s>>>(src64, imgs, H, W, C, k, p, dst, ld);
        return cudaGetLastError();
    }
    if (src64) im2col_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(src64, imgs, H, W, C, k, p, dst, ld);
    else im2col_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(src32, imgs, H, W, C, k, p, dst, ld);
    return cudaGetLastError();
}

cudaError_t launch_im2col_act(const float* x, int imgs, int hp, int wp, long long ldx, int C, int k, int Ho, int Wo,
                              float* dst, long long ldc, cudaStream_t s, int stride) {
    const long long n = static_cast<long long>(imgs) * Ho * Wo * ldc;
    if (n <= 0) return cudaSuccess;
    if (C % 4 == 0 && ldx % 4 == 0 && ldc % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
        reinterpret_cast<uintptr_t>(dst) % 16 == 0) {
        const long long nv = static_cast<long long>(imgs) * Ho * Wo * k * k * (C / 4);
        if (nv < (1LL << 31))
            pdl_launch(im2col_act_vec_kernel<unsigned>, dim3(grid_for(nv, 256)), dim3(256), 0, s, x, imgs, hp, wp, ldx,
                       C, k, Ho, Wo, dst, ldc, stride);
        else
            pdl_launch(im2col_act_vec_kernel<long long>, dim3(grid_for(nv, 256)), dim3(256), 0, s, x, imgs, hp, wp,
                       ldx, C, k, Ho, Wo, dst, ldc, stride);
        return cudaGetLastError();
    }
    pdl_launch(im2col_act_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, x, imgs, hp, wp, ldx, C, k, Ho, Wo, dst, ldc,
               stride);
    return cudaGetLastError();
}

cudaError_t launch_col2im(const float* dcols, long long ldk, int imgs, int H, int W, int C, int k, int p, int c0,
                          int nc, float* dst, long long ldo, cudaStream_t s, int stride) {
    const long long n = static_cast<long long>(imgs) * H * W * nc;
    if (n <= 0) return cudaSuccess;
    const int Ho = (H + 2 * p - k) / stride + 1, Wo = (W + 2 * p - k) / stride + 1;
    if (C % 4 == 0 && c0 % 4 == 0 && nc % 4 == 0 && ldk % 4 == 0 && ldo % 4 == 0 &&
        reinterpret_cast<uintptr_t>(dcols) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0) {
        const long long nv = n / 4;
        if (k == 3 && stride == 2) {
            const int grid = grid_for(nv, 256);
            if (nv + 2LL * grid * 256 < (1LL << 31))
                pdl_launch(col2im_k3s2_kernel<unsigned>, dim3(grid), dim3(256), 0, s, dcols, ldk, imgs, H, W, C, p, Ho,
                           Wo, c0, nc, dst, ldo);
            else
                pdl_launch(col2im_k3s2_kernel<long long>, dim3(grid), dim3(256), 0, s, dcols, ldk, imgs, H, W, C, p,
                           Ho, Wo, c0, nc, dst, ldo);
            return cudaGetLastError();
        }
        if (k == 3) {
            if (nv < (1LL << 31))
                pdl_launch(col2im_k3_kernel<unsigned>, dim3(grid_for(nv, 256)), dim3(256), 0, s, dcols, ldk, imgs, H, W,
                           C, p, Ho, Wo, c0, nc, dst, ldo, stride);
            else
                pdl_launch(col2im_k3_kernel<long long>, dim3(grid_for(nv, 256)), dim3(256), 0, s, dcols, ldk, imgs, H,
                           W, C, p, Ho, Wo, c0, nc, dst, ldo, stride);
            return cudaGetLastError();
        }
        if (nv < (1LL << 31))
            pdl_launch(col2im_vec_kernel<unsigned>, dim3(grid_for(nv, 256)), dim3(256), 0, s, dcols, ldk, imgs, H, W, C,
                       k, p, Ho, Wo, c0, nc, dst, ldo, stride);
        else
            pdl_launch(col2im_vec_kernel<long long>, dim3(grid_for(nv, 256)), dim3(256), 0, s, dcols, ldk, imgs, H, W,
                       C, k, p, Ho, Wo, c0, nc, dst, ldo, stride);
        return cudaGetLastError();
    }
    pdl_launch(col2im_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, dcols, ldk, imgs, H, W, C, k, p, Ho, Wo, c0, nc, dst, ldo,
               stride);
    return cudaGetLastError();
}

cudaError_t launch_dense_conv_expand(const DenseConvGeom& g, const float* W, float* Wx, cudaStream_t s) {
    const long long n = static_cast<long long>(g.u) * g.C;
    if (n <= 0) return cudaSuccess;
    dense_conv_expand_kernel<<<grid_for(n, 256), 256, 0, s>>>(g, W, Wx);
    return cudaGetLastError();
}

cudaError_t launch_dense_conv_fold_sgd(const DenseConvGeom& g, const float* dWx, float* W, float* Wx,
                                       const double* alpha, float inv_b, int* flag, cudaStream_t s,
                                       const float* bpart, int bchunks, float* bias) {
    const long long n = static_cast<long long>(g.u) * g.C;
    if (n <= 0) return cudaSuccess;
    if (g.k == 3 && g.pad == 1 && g.H == 2 && g.W == 2 && g.Ho == 2 && g.Wo == 2) {
        const unsigned blocks = static_cast<unsigned>((n + 255) / 256) + (bias != nullptr ? (g.u + 7) / 8 : 0);
        pdl_launch(dense_conv_update_2x2_kernel, dim3(blocks), dim3(256), 0, s, g, dWx, W, Wx, alpha, inv_b, flag, bpart, bchunks, bias);
        return cudaGetLastError();
    }
    if (bias != nullptr) {
        cudaError_t e = launch_bias_from_partials(bpart, bchunks, g.u, bias, alpha, inv_b, s);
        if (e != cudaSuccess) return e;
    }
    pdl_launch(dense_conv_fold_sgd_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, g, dWx, W, Wx, alpha, inv_b, flag);
    return cudaGetLastError();
}

// Keeps a stream busy for ~`ns` nanoseconds (profiling: the ops that follow
// are already enqueued when it finishes, so their start events carry no
// host-launch latency).
__global__ void spin_kernel(long long ns) {
    const long long t0 = clock64();
    const long long cycles = ns * 2;  // >= ns at <= 2 GHz
    while (clock64() - t0 < cycles) {
    }
}

cudaError_t launch_spin(long long ns, cudaStream_t s) {
    spin_kernel<<<1, 32, 0, s>>>(ns);
    return cudaGetLastError();
}

cudaError_t launch_pad_input(const double* src64, const float* src32, int imgs, int H, int W, int C, float* dst,
                             int p, long long ld, cudaStream_t s) {
    const long long n = static_cast<long long>(imgs) * H * W * C;
    if (n <= 0) return cudaSuccess;
    if (src64) pad_input_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(src64, imgs, H, W, C, dst, p, ld);
    else pad_input_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(src32, imgs, H, W, C, dst, p, ld);
    return cudaGetLastError();
}

bool vec4_ok(long long a, long long b = 0, long long c = 0) { return a % 4 == 0 && b % 4 == 0 && c % 4 == 0; }

int group_block(int groups) {
    // a multiple of `groups` near 256 threads
    int b = groups >= 256 ? groups : (256 / groups) * groups;
    return b > 1024 ? groups : b;
}

cudaError_t launch_pool_fwd(const float* U, long long ldu, int imgs, int Ho, int Wo, int uch, int pool,
                            unsigned char* argmax, const ActLayout& out, const PoolDsts& dsts, cudaStream_t s) {
    const long long n = static_cast<long long>(imgs) * (Ho / pool) * (Wo / pool) * uch;
    if (n <= 0) return cudaSuccess;
    bool v4 = vec4_ok(uch, ldu) && (out.kind != 0 || vec4_ok(out.ld, out.col0)) &&
              reinterpret_cast<uintptr_t>(U) % 16 == 0;
    for (int d = 0; d < dsts.n; ++d) v4 = v4 && reinterpret_cast<uintptr_t>(dsts.ptr[d]) % 16 == 0;
    const bool i32 = n < (1LL << 31);
    if (v4) {
        if (i32) pdl_launch(pool_fwd_kernel<4, unsigned>, dim3(grid_for(n / 4, 256)), dim3(256), 0, s, U, ldu, imgs, Ho, Wo, uch, pool, argmax, out, dsts);
        else pdl_launch(pool_fwd_kernel<4, long long>, dim3(grid_for(n / 4, 256)), dim3(256), 0, s, U, ldu, imgs, Ho, Wo, uch, pool, argmax, out, dsts);
    } else {
        if (i32) pdl_launch(pool_fwd_kernel<1, unsigned>, dim3(grid_for(n, 256)), dim3(256), 0, s, U, ldu, imgs, Ho, Wo, uch, pool, argmax, out, dsts);
        else pdl_launch(pool_fwd_kernel<1, long long>, dim3(grid_for(n, 256)), dim3(256), 0, s, U, ldu, imgs, Ho, Wo, uch, pool, argmax, out, dsts);
    }
    return cudaGetLastError();
}

int conv_merge_blocks() { return 148 * 4; }

cudaError_t launch_conv_merge(const ConvMerge& m, float* db_partial, cudaStream_t s) {
    const long long n = static_cast<long long>(m.imgs) * m.Ho * m.Wo * m.uch;
    bool v4 = m.slot_kind == 0 && vec4_ok(m.uch, m.lds, m.ldd) && (m.mask_kind != 1 || vec4_ok(m.ldu)) &&
              ((m.mask_kind != 2 && m.mask_kind != 3) || vec4_ok(m.act_layout.ld, m.act_layout.col0)) &&
              reinterpret_cast<uintptr_t>(m.d_pad) % 16 == 0;
    for (int k = 0; k < m.slots.n; ++k) v4 = v4 && reinterpret_cast<uintptr_t>(m.slots.slot[k]) % 16 == 0;
    const int vec = v4 ? 4 : 1;
    const int groups = m.uch / vec;
    const int block = group_block(groups);
    const int grid = conv_merge_blocks();
    const size_t shmem = sizeof(float) * block * vec;
    if (n <= 0) {
        return cudaMemsetAsync(db_partial, 0, sizeof(float) * grid * m.uch, s);
    }
    const bool i32 = n < (1LL << 31);
    if (v4 && (m.pool == 1 || m.pool == 2)) {
        pdl_launch(conv_merge_rows_kernel<2>, dim3(grid), dim3(block), shmem, s, m, db_partial);
    } else if (v4) {
        if (i32) pdl_launch(conv_merge_kernel<4, unsigned>, dim3(grid), dim3(block), shmem, s, m, db_partial);
        else pdl_launch(conv_merge_kernel<4, long long>, dim3(grid), dim3(block), shmem, s, m, db_partial);
    } else {
        if (i32) pdl_launch(conv_merge_kernel<1, unsigned>, dim3(grid), dim3(block), shmem, s, m, db_partial);
        else pdl_launch(conv_merge_kernel<1, long long>, dim3(grid), dim3(block), shmem, s, m, db_partial);
    }
    return cudaGetLastError();
}

cudaError_t launch_unpack_gather(const float* recv, int g, int rows, int u, float* dst, long long ld, cudaStream_t s) {
    const long long n = static_cast<long long>(g) * rows * u;
    if (n <= 0) return cudaSuccess;
    pdl_launch(unpack_gather_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, recv, g, rows, u, dst, ld);
    return cudaGetLastError();
}

cudaError_t launch_residual_act(float* U, long long ldu, int imgs, int Ho, int Wo, int uch, int c0, int relu,
                                int pool, const SkipSrc& skip, const ActLayout& out, const PoolDsts& dsts,
                                cudaStream_t s) {
    const long long n = static_cast<long long>(imgs) * (Ho / pool) * (Wo / pool) * (uch / 4);
    if (n <= 0) return cudaSuccess;
    if (uch % 4 != 0 || ldu % 4 != 0 || (out.kind == 0 && (out.ld % 4 != 0 || out.col0 % 4 != 0)))
        return cudaErrorInvalidValue;
    const int write_u = !(relu && pool == 1);  // relu(u) > 0 <=> u > 0: the mask can read the activation
    const int skip_vec = skip.lay.ld % 4 == 0 && c0 % 4 == 0 && reinterpret_cast<uintptr_t>(skip.a) % 16 == 0;
    pdl_launch(residual_act_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, U, ldu, imgs, Ho, Wo, uch, c0, relu, pool,
               skip, out, dsts, write_u, skip_vec);
    return cudaGetLastError();
}

cudaError_t launch_conv_merge_res(const ConvMerge& m, int pool_avg, const SkipGrad& sg, float* db_partial,
                                  cudaStream_t s) {
    const int grid = conv_merge_blocks();
    if (m.uch % 4 != 0 || m.slot_kind != 0 || !vec4_ok(m.lds, m.ldd) || (sg.d != nullptr && !vec4_ok(sg.ldd, sg.c0)))
        return cudaErrorInvalidValue;
    const int groups = m.uch / 4;
    const int block = group_block(groups);
    if (static_cast<long long>(m.imgs) * m.Ho * m.Wo * m.uch <= 0)
        return cudaMemsetAsync(db_partial, 0, sizeof(float) * grid * m.uch, s);
    pdl_launch(conv_merge_res_kernel<false>, dim3(grid), dim3(block), sizeof(float) * block * 4, s, m, pool_avg, sg,
               Col2imSrc{}, db_partial);
    return cudaGetLastError();
}

cudaError_t launch_conv_merge_res_col2im(const ConvMerge& m, int pool_avg, const SkipGrad& sg, const Col2imSrc& cx,
                                         float* db_partial, cudaStream_t s) {
    const int grid = conv_merge_blocks();
    if (m.uch % 4 != 0 || m.pool != 1 || !vec4_ok(m.ldd, 0) || (sg.d != nullptr && !vec4_ok(sg.ldd, sg.c0)) ||
        cx.dcols == nullptr || cx.C % 4 != 0 || cx.c0 % 4 != 0 || cx.ldk % 4 != 0 ||
        reinterpret_cast<uintptr_t>(cx.dcols) % 16 != 0)
        return cudaErrorInvalidValue;
    const int groups = m.uch / 4;
    const int block = group_block(groups);
    if (static_cast<long long>(m.imgs) * m.Ho * m.Wo * m.uch <= 0)
        return cudaMemsetAsync(db_partial, 0, sizeof(float) * grid * m.uch, s);
    pdl_launch(conv_merge_res_kernel<true>, dim3(grid), dim3(block), sizeof(float) * block * 4, s, m, pool_avg, sg, cx,
               db_partial);
    return cudaGetLastError();
}

cudaError_t launch_bias_from_partials(const float* partial, int chunks, int u, float* bias, const double* alpha,
                                      float inv_b, cudaStream_t s) {
    if (u <= 0) return cudaSuccess;
    pdl_launch(bias_update_cols_kernel, dim3((u + 31) / 32), dim3(dim3(32, 32)), 0, s, partial, u, chunks, bias, alpha, inv_b);
    return cudaGetLastError();
}

cudaError_t launch_finalize(StepState* st, const double* loss_row, const int* correct_row, int b,
                            double* loss_hist, double* acc_hist, int hist_cap, int write_hist,
                            cudaStream_t s) {
    pdl_launch(finalize_kernel, dim3(1), dim3(kRowThreads), 0, s, st, loss_row, correct_row, b, loss_hist, acc_hist,
                                              hist_cap, write_hist);
    return cudaGetLastError();
}

}  // namespace ppb
