// Halo-reuse weight gradient of a 3x3 / stride-1 / pad-1 convolution with 64
// input and 64 output channels (VGG conv2, the ResNet-18 stage-1 convs), for
// sm_100a (tcgen05, TF32).
//
//   dW^T[(r*3 + s)*64 + c][o] = sum_p  x_pad[p + (r, s)][c] * delta[p][o]
//
// The generic path (tc_gemm_kernel, OP_CONV_KPIX operands) splits the 576
// output rows into 5 M tiles and, per 32-pixel K block, TMA-loads the 9 taps'
// shifted input boxes again for every tile: 24 KB per 4 MMAs of N = 64, about
// twice what the TMA unit delivers per MMA time, so the tensor core idled.
//
// Here one CTA owns ALL 576 rows (six 64-column TMEM accumulators) for a
// contiguous range of K blocks (split-K over the batch: one split per CTA).
// Per K block (32 output pixels of one image row) it loads the input rows
// h-1..h+1 as six {32 channels x 34 pixels} boxes -- [row tap r][channel
// block] in 5 KB slots -- plus the error signal's two {32 x 32} boxes, 34 KB
// in all.  The MN-major A operand of tap (r, s) is the slot of (r, block)
// started s pixel rows (s * 128 B) in: with slots 5 KB apart (the descriptor's
// leading byte offset) one M = 128 MMA covers atoms (r0, c0..31), (r0,
// c32..63), (r1, ...), (r1, ...), a second covers (r2, ...) plus two atoms
// past the stage whose rows are discarded.  24 MMAs (128 x 64 x 8) per 34 KB
// loaded: MMA-bound instead of TMA-bound.  The swizzle phase follows the
// absolute shared-memory address as the TMA wrote it (the same property the
// halo forward kernel relies on for its row shifts).
//
//   warp 0      TMA producer (one thread)
//   warp 1      MMA issuer (one thread)
//   warp 2      TMEM allocator (512 columns)
//   warps 4..7  a previous wgrad's split-K reduction + SGD (side job) while
//               the mainloop runs, then the epilogue: the CTA's 576 x 64 partial sums -> split-K
//               workspace slice blockIdx.x (the existing ordered reduction /
//               side job then sums the slices and applies SGD)
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "dev_knobs.h"
#include "gemm_tc_kernel.cuh"  // run_side_job

namespace ppb {

namespace {

std::atomic<unsigned> g_wg_attr{0};

constexpr int kWgThreads = 256;
constexpr int kABox = 34 * 128;        // {32 ch, 34 px} input box
constexpr int kASlot = 5 * 1024;       // its 1 KB-aligned slot (SW128 boxes)
constexpr int kAStage = 6 * kASlot;    // [r][channel block]
constexpr int kBBox = 32 * 128;        // {32 out-ch, 32 px} error-signal box
constexpr int kStage = kAStage + 2 * kBBox;
constexpr int kSlack = 4096;           // the padding atoms of the r = 2 MMA read past the last stage
constexpr int kTx = 6 * kABox + 2 * kBBox;
constexpr int kMaxStages = 5;
constexpr int kSmem = 1024 + kMaxStages * kStage + kSlack + 256;

__global__ void __launch_bounds__(kWgThreads, 1)
    wgrad_halo_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      const __grid_constant__ WgradGeom g, const __grid_constant__ SplitK sk,
                      const __grid_constant__ SideJob sj) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    constexpr int nst = kMaxStages;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + nst * kStage + kSlack);
    uint64_t* empty = full + nst;
    uint64_t* done = empty + nst;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int warp = threadIdx.x / 32;
    const int kb0 = static_cast<int>(static_cast<long long>(blockIdx.x) * g.kbs / gridDim.x);
    const int kb1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * g.kbs / gridDim.x);

    if (warp == 0 && elect_one()) {
        tma_prefetch(&ta);
        tma_prefetch(&tb);
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_wait();

    if (warp == 0) {
        if (elect_one()) {
            const int wblocks = g.wo / 32;
            int stage = 0;
            uint32_t phase = 0;
            int img = kb0 / (g.ho * wblocks);
            int rem = kb0 - img * g.ho * wblocks;
            int h = rem / wblocks, wb = rem - h * wblocks;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full[stage], kTx);
                uint8_t* st = ring + stage * kStage;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int cb = 0; cb < 2; ++cb)
                        tma_load_4d(st + (r * 2 + cb) * kASlot, &ta, &full[stage], cb * 32, wb * 32, h + r, img);
#pragma unroll
                for (int ob = 0; ob < 2; ++ob)
                    tma_load_4d(st + kAStage + ob * kBBox, &tb, &full[stage], ob * 32, wb * 32 + g.q, h + g.q, img);
                if (++wb == wblocks) {
                    wb = 0;
                    if (++h == g.ho) {
                        h = 0;
                        ++img;
                    }
                }
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        __syncwarp();
        griddep_launch_dependents();
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t idesc = idesc_tf32(64, true, true, 128);
            // MN-major (SW128_BASE32B): K8 step = 8 pixel rows (1 KB), 4-row K
            // groups 512 B apart; A atoms one slot apart, B atoms one box apart
            const uint64_t a0 = umma_desc<kLayoutSW128Base32>(smem_u32(ring), kASlot, 512);
            const uint64_t b0 = umma_desc<kLayoutSW128Base32>(smem_u32(ring + kAStage), kBBox, 512);
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint64_t ad = desc_advance(a0, stage * kStage);
                const uint64_t bd = desc_advance(b0, stage * kStage);
#pragma unroll
                for (int s = 0; s < 3; ++s) {
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const uint32_t d_tmem = tmem_base + (s * 2 + t) * 64;
                        const uint64_t at = desc_advance(ad, t * 4 * kASlot + s * 128);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_tf32(d_tmem, desc_advance(at, kk * 1024), desc_advance(bd, kk * 1024), idesc,
                                     (kb != kb0 || kk != 0) ? 1u : 0u);
                    }
                }
                mma_commit(&empty[stage]);
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            mma_commit(done);
        }
        __syncwarp();
    } else if (warp >= 4) {
        // epilogue: accumulator (s, t), TMEM lane quarter q = rows q*32..q*32+31
        // of the tile: t = 0 -> row tap r = q / 2, t = 1 -> r = 2 (q < 2 only)
        const int q = warp & 3;
        const int lane = threadIdx.x & 31;
        if (sj.on)
            run_side_job(sj, static_cast<long long>(blockIdx.x) * 128 + (threadIdx.x - 128),
                         static_cast<long long>(gridDim.x) * 128, lane);
        mbar_wait(done, 0);
        tc_fence_after();
        float* ws = sk.ws + static_cast<long long>(blockIdx.x) * sk.stride;
#pragma unroll 1
        for (int acc = 0; acc < 6; ++acc) {
            const int s = acc >> 1, t = acc & 1;
            if (t == 1 && q >= 2) continue;  // padding atoms
            const int r = t == 0 ? (q >> 1) : 2;
            const int m = (r * 3 + s) * 64 + (q & 1) * 32 + lane;
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * 64 + nb * 32, v);
                tmem_ld_wait();
                if (sk.trans) {  // [n][m]: for each column the lanes write 32 consecutive m
#pragma unroll
                    for (int i = 0; i < 32; ++i) ws[static_cast<long long>(nb * 32 + i) * sk.ld + m] = __uint_as_float(v[i]);
                } else {
                    float4* row = reinterpret_cast<float4*>(ws + static_cast<long long>(m) * sk.ld + nb * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        row[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace

// A: the input activation as the tc path's OP_CONV_KPIX operand (3x3 taps,
// 64 channels, no offset: stride 1, pad 1); B: the error signal (one tap, 64
// channels, ring offset q); 576 x 64 output, wgrad + SGD without per-micro-
// batch slices.
bool wgrad_halo_eligible(const GemmDesc& d) {
    if (d.epi.mode != EPI_SGD || d.partial_out || d.force_splits > 0) return false;
    if (!d.a.mn_major || !d.b.mn_major) return false;
    const ConvGeom& ga = d.a.geom;
    const ConvGeom& gb = d.b.geom;
    if (ga.mode != OP_CONV_KPIX || ga.ksz != 3 || ga.off != 0 || ga.ck != 64 || d.a.ch != 64) return false;
    if (gb.mode != OP_CONV_KPIX || gb.ksz != 1 || d.b.ch != 64) return false;
    if (d.M != 576 || d.N != 64) return false;
    const int wo = ga.wo, ho = ga.ho;
    if (wo % 32 != 0 || d.a.wp != wo + 2 || d.a.hp != ho + 2) return false;
    if (gb.wo != wo || gb.ho != ho || d.b.wp != wo + 2 * gb.off || d.b.hp != ho + 2 * gb.off) return false;
    if (static_cast<long long>(d.a.imgs) * ho * wo != d.K) return false;
    if (d.a.ld % 4 != 0 || d.b.ld % 4 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(d.a.ptr) & 15u) != 0 || (reinterpret_cast<uintptr_t>(d.b.ptr) & 15u) != 0)
        return false;
    return !dev_knob("PPB_NO_WGRAD_HALO");  // A/B switch (DEV builds)
}

bool wgrad_halo_prepare(const GemmDesc& d, TcGemmPlan* out, char* err, size_t errlen, const WsAlloc& ws_alloc) {
    if (!ws_alloc) {
        snprintf(err, errlen, "halo wgrad needs a split-K workspace");
        return false;
    }
    TcGemmPlan p;
    p.halo = 2;
    p.M = d.M;
    p.N = d.N;
    p.K = d.K;
    p.a_mn = p.b_mn = true;
    p.bn = 64;
    p.cg = 1;
    p.epi = d.epi;
    p.epi.M = d.M;
    p.epi.N = d.N;
    p.ga = d.a.geom;
    p.gb = d.b.geom;
    WgradGeom& g = p.wg;
    g.wo = d.a.geom.wo;
    g.ho = d.a.geom.ho;
    g.q = d.b.geom.off;
    g.kbs = static_cast<int>(d.K / 32);
    const int sms = sm_count();
    p.grid = g.kbs < sms ? g.kbs : sms;  // every CTA owns >= 1 K block
    p.sk.splits = p.grid;
    p.sk.kps = 1;
    p.sk.trans = d.epi.sgd_t ? 1 : 0;
    p.sk.ld = p.sk.trans ? (d.M + 3) / 4 * 4 : (d.N + 3) / 4 * 4;
    p.sk.stride = p.sk.ld * (p.sk.trans ? d.N : d.M);
    p.sk.ws = ws_alloc(static_cast<size_t>(p.sk.stride) * p.sk.splits);
    if (p.sk.ws == nullptr) {
        snprintf(err, errlen, "split-K workspace allocation failed");
        return false;
    }
    Operand a = d.a;
    a.geom.bw = 34;  // {32 ch, 34 px, 1 row, 1 image}
    a.geom.bh = 1;
    a.geom.bn = 1;
    a.geom.mode = OP_CONV_KPIX;
    Operand b = d.b;
    b.geom.bw = 32;
    b.geom.bh = 1;
    b.geom.bn = 1;
    if (!encode_conv_map(&p.ta, a, err, errlen) || !encode_conv_map(&p.tb, b, err, errlen)) return false;
    *out = p;
    return true;
}

cudaError_t wgrad_halo_launch(const TcGemmPlan& p, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    if ((g_wg_attr.load() & (1u << (dev & 31))) == 0) {
        const cudaError_t e = cudaFuncSetAttribute(wgrad_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        g_wg_attr.fetch_or(1u << (dev & 31));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(kWgThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, wgrad_halo_kernel, p.ta, p.tb, p.wg, p.sk, p.sj);
    if (e != cudaSuccess || p.sk.fixup || p.sk.deferred || p.sk.partial) return e;
    return tc_gemm_launch_reduce(p, s);
}

}  // namespace ppb
