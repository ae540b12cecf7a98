// Persistent, warp-specialised tcgen05 TF32 GEMM for sm_100a.
//
//   warps 0, 3  : TMA producers (one elected lane each: A, B), SWIZZLE_128B tiles
//                 into a kStages-deep shared-memory ring guarded by full/empty
//                 mbarriers (full: one arrival per producer)
//   warp 1      : MMA issuer (one elected lane of the leader CTA):
//                 tcgen05.mma.cta_group::{1,2}.kind::tf32, accumulator in TMEM
//   warp 2      : TMEM allocator (2 x BN columns: double-buffered accumulator)
//   warps 4..7  : epilogue: tcgen05.ld -> registers -> fused epilogue -> global
//
// CG = 1: one CTA computes a 128 x BN tile (UMMA M = 128).
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
//         UMMA M = 256: each CTA stages its own 128 rows of A and half of the
//         BN rows of B, so each SM reads half the operand bytes per FLOP; the
//         leader CTA issues the MMAs for both and its commits multicast to
//         the pair's barriers.
//
// BK = 32 fp32 (one 128-byte swizzle atom for K-major operands).  K-major
// operands are loaded as one TMA box {32 (K), rows}; MN-major operands as
// rows/32 boxes {32 (MN), 32 (K)}, each a 4 KB SW128_BASE32B atom column.
// See gemm.h for how the forward / dgrad / wgrad products of the partitioned
// step map onto A and B.
//
// This header holds the kernels; each (A_MN, B_MN) operand-major combination
// is instantiated in its own translation unit (gemm_tc_inst_*.cu) so the
// 24 kernel instantiations compile in parallel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "dev_knobs.h"
#include "dense_conv.cuh"
#include "epilogue.cuh"
#include "gemm_tc.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace ppb {

namespace {

constexpr int kThreads = 128 + 32 * kEpiWarps;  // 4 control warps + epilogue warps

template <int BN, int CG>
struct TcCfg {
    static constexpr int kBNc = BN / CG;  // rows of B staged per CTA
    static constexpr int kStageA = kBM * kBK * 4;  // bytes
    static constexpr int kStageB = kBNc * kBK * 4;
    static constexpr int kStageBytes = kStageA + kStageB;
    static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
    // accumulator ring: 4 deep up to BN = 128 (512 TMEM columns at most), 2 at
    // BN = 256; by-tile epilogues give each warp group every other accumulator
    static constexpr int kAcc = BN <= 128 ? 4 : 2;
    static constexpr int kTmemCols = kAcc * BN;
};

// One split-K work item (row r, columns c4..c4+3 of the workspace): sum the
// splits in order 0..splits-1, then the GEMM's epilogue (SGD on dW^T / dW).
__device__ __forceinline__ void splitk_item_seq(const EpiParams& epi, const SplitK& sk, int M, int N, long long item) {
    const int R = sk.trans ? N : M;
    const int Cc = sk.trans ? M : N;
    const int cq = (Cc + 3) / 4;
    if (item >= static_cast<long long>(R) * cq) return;
    const int r = static_cast<int>(item / cq);
    const int c4 = static_cast<int>(item - static_cast<long long>(r) * cq) * 4;
    const int nc = Cc - c4 < 4 ? Cc - c4 : 4;
    const bool vec = nc == 4 && (sk.ld & 3) == 0;
    const long long off = static_cast<long long>(r) * sk.ld + c4;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    // association of splitk_epilogue_kernel: sequential for < 16 splits;
    // otherwise 8 phase sums (splits p, p+8, ...) added in phase order
    const int nph = sk.splits >= 64 ? 32 : sk.splits >= 16 ? 8 : 1;
#pragma unroll 1
    for (int ph = 0; ph < nph; ++ph) {
        float b[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int sp = ph; sp < sk.splits; sp += nph) {
            const float* src = sk.ws + static_cast<long long>(sp) * sk.stride + off;
            if (vec) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(src));
                b[0] += t.x;
                b[1] += t.y;
                b[2] += t.z;
                b[3] += t.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < nc) b[j] += __ldcg(src + j);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] += b[j];
    }
    if (sk.trans) {
        const float alpha = static_cast<float>(*epi.alpha);
        float* w = epi.W + static_cast<long long>(r) * epi.ldw + c4;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j < nc) {
                const float g = a[j] * epi.inv_b;
                bad |= !isfinite(g);
                w[j] -= alpha * g;
            }
        }
        if (bad && epi.flag != nullptr) atomicOr(epi.flag, 1);
        return;
    }
    const long long row_off = epi.mode == EPI_STORE ? epi_store_row(epi, r) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < nc) epilogue1(epi, r, c4 + j, a[j], row_off);
}

// The side job over every epilogue thread of the grid (gt = global epilogue
// thread index, nt = their count).  Bias job first: warp-group of 32 lanes =
// 4 columns x 8 phases (phase p sums chunks p, p+8, ... in order), butterfly
// over the phases (fixed tree), lane with phase 0 updates the column.
// Sum of bpart[k * bu + col] over k = k0, k0 + 8, ... < chunks, added in
// ascending k (the bias-gradient partials' fixed order) with eight loads in
// flight per batch: the one-load-per-add loop the compiler emitted for the
// plain form was a serial chain of L2 round trips (~74 per lane for a
// 592-chunk merge), the longest part of conv1's wgrad side job.
__device__ __forceinline__ float bias_chunk_sum(const float* __restrict__ bpart, int bu, int col, int k0, int chunks) {
    float acc = 0.f;
    int k = k0;
    for (; k + 7 * 8 < chunks; k += 64) {
        float t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = __ldcg(bpart + static_cast<long long>(k + 8 * i) * bu + col);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += t[i];
    }
    for (; k < chunks; k += 8) acc += __ldcg(bpart + static_cast<long long>(k) * bu + col);
    return acc;
}

__device__ __forceinline__ void run_side_job(const SideJob& sj, long long gt, long long nt, int lane) {
    const SplitK& sk = sj.sk;
    if (sk.bias != nullptr) {
        const long long gw = gt >> 5, nw = nt >> 5;
        const int groups = (sk.bu + 3) / 4;
        for (long long grp = gw; grp < groups; grp += nw) {
            const int col = static_cast<int>(grp) * 4 + (lane >> 3), ph = lane & 7;
            const float acc0 = col < sk.bu ? bias_chunk_sum(sk.bpart, sk.bu, col, ph, sk.bchunks) : 0.f;
            float acc = acc0;
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            if (ph == 0 && col < sk.bu) sk.bias[col] -= static_cast<float>(*sj.epi.alpha) * (acc * sj.epi.inv_b);
        }
    }
    if (sj.kind == 1) {  // dense-conv fold + SGD + re-expansion, one (co, ci) pair per item
        DenseConvGeom g;
        g.u = sj.dc_u;
        g.C = sj.dc_C;
        g.ck = sj.dc_ck;
        g.ldw = sj.dc_ldw;
        g.ldx = sj.dc_ldx;
        const float a = static_cast<float>(*sj.epi.alpha);
        const long long items = static_cast<long long>(g.u) * g.C;
        for (long long it = gt; it < items; it += nt)
            dense_conv_update_2x2_item(g, sj.dWx, sj.Wm, sj.Wx, a, sj.epi.inv_b, sj.epi.flag, it);
        return;
    }
    const long long R = sk.trans ? sj.N : sj.M, Cc = sk.trans ? sj.M : sj.N;
    const int cq = static_cast<int>((Cc + 3) / 4);
    const long long items = R * cq;
    // 4 items per thread per pass (independent load chains: each thread owns
    // ~items / nt of them, so one-at-a-time would be latency-bound); full
    // float4 items only, the ragged ones go through splitk_item_seq
    const int nph = sk.splits >= 64 ? 32 : sk.splits >= 16 ? 8 : 1;
    const bool vec_ok = (sk.ld & 3) == 0 && (Cc & 3) == 0 && !sj.scalar;
    long long it = gt;
    if (vec_ok) {
        for (; it + 3 * nt < items; it += 4 * nt) {
            float4 a[4];
            long long off[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const long long t = it + i * nt;
                const long long r = t / cq;
                off[i] = r * sk.ld + (t - r * cq) * 4;
                a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll 1
            for (int ph = 0; ph < nph; ++ph) {
                float4 b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
                for (int sp = ph; sp < sk.splits; sp += nph) {
                    const float* base = sk.ws + static_cast<long long>(sp) * sk.stride;
                    float4 t[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) t[i] = __ldcg(reinterpret_cast<const float4*>(base + off[i]));
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        b[i].x += t[i].x;
                        b[i].y += t[i].y;
                        b[i].z += t[i].z;
                        b[i].w += t[i].w;
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a[i].x += b[i].x;
                    a[i].y += b[i].y;
                    a[i].z += b[i].z;
                    a[i].w += b[i].w;
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const long long t = it + i * nt;
                const int r = static_cast<int>(t / cq);
                const int c4 = static_cast<int>(t - static_cast<long long>(r) * cq) * 4;
                const float av[4] = {a[i].x, a[i].y, a[i].z, a[i].w};
                if (sk.trans) {
                    const float alpha = static_cast<float>(*sj.epi.alpha);
                    float* w = sj.epi.W + static_cast<long long>(r) * sj.epi.ldw + c4;
                    bool bad = false;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float g = av[j] * sj.epi.inv_b;
                        bad |= !isfinite(g);
                        w[j] -= alpha * g;
                    }
                    if (bad && sj.epi.flag != nullptr) atomicOr(sj.epi.flag, 1);
                } else {
                    const long long row_off = sj.epi.mode == EPI_STORE ? epi_store_row(sj.epi, r) : 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) epilogue1(sj.epi, r, c4 + j, av[j], row_off);
                }
            }
        }
    }
    for (; it < items; it += nt) splitk_item_seq(sj.epi, sk, sj.M, sj.N, it);
}

template <bool A_MN, bool B_MN, int BN, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   int M, int N, int K, const __grid_constant__ EpiParams epi,
                   const __grid_constant__ ConvGeom ga, const __grid_constant__ ConvGeom gb,
                   const __grid_constant__ SplitK sk, const __grid_constant__ TmaStore ts, int nst,
                   const __grid_constant__ SideJob sj) {
    using C = TcCfg<BN, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    // row reuse (ga.rr, 3x3 implicit conv over whole image rows): one A box of
    // bh + ksz - 1 image rows serves the ksz row taps of one (column tap,
    // channel block) pair, so a stage holds that box and ksz B blocks
    const int tps = ga.rr ? ga.ksz : 1;                                        // K blocks per stage
    const int stA = ga.rr ? (ga.bh + ga.ksz - 1) * ga.bw * 128 : C::kStageA;  // bw % 8 == 0: 1 KB multiple
    const int stB = tps * C::kStageB;
    uint8_t* sA = smem;
    uint8_t* sB = smem + nst * stA;  // nst ring stages (host: smem budget)
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + nst * (stA + stB));
    uint64_t* empty_bar = full_bar + nst;
    uint64_t* tfull_bar = empty_bar + nst;       // [kAcc]
    uint64_t* tempty_bar = tfull_bar + C::kAcc;  // [kAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + C::kAcc);
    float* db_s = reinterpret_cast<float*>(smem + nst * (stA + stB) + 256);  // [4][ldb] (EPI_MERGE db)
    uint8_t* stg = smem + nst * (stA + stB) + ts.stage_off;                  // TMA-store staging

    const int warp = threadIdx.x / 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    constexpr int TM = kBM * CG;  // tile rows
    const int num_m = (M + TM - 1) / TM;
    const int num_n = (N + BN - 1) / BN;
    const int num_mn = num_m * num_n;
    const int num_tiles = num_mn * sk.splits;  // split-K: tile = (split, n, m)
    const int nk = (K + kBK - 1) / kBK;
    const int unit = blockIdx.x / CG;  // cluster (or CTA) index
    const int units = gridDim.x / CG;

    if (warp == 0 && elect_one()) {
        tma_prefetch(&ta);
        tma_prefetch(&tb);
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full_bar[s], 2);  // the A and the B producer each arrive (with their tx bytes)
            mbar_init(&empty_bar[s], 1);
        }
        for (int i = 0; i < C::kAcc; ++i) {  // nst <= 8: 2 * 8 + 2 * 4 barriers + slot fit the 256 B block
            mbar_init(&tfull_bar[i], 1);
            mbar_init(&tempty_bar[i], kEpiWarps * CG);  // one arrival per epilogue warp of the pair
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        if (CG == 2) tmem_alloc_pair(tmem_slot, C::kTmemCols);
        else tmem_alloc(tmem_slot, C::kTmemCols);
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // prologue done (barriers, TMEM, tensor-map prefetch): wait for the
    // stream predecessor's results (the successor is released after the last
    // MMA is issued, so its waiting CTAs do not squat on SMs other streams use)
    griddep_wait();

    // ------------------------------------------------ TMA producers: warp 0 stages A, warp 3 stages B
    // (two single-thread issue streams: one thread's per-K-block bookkeeping
    // was on the critical path of the N = 256 pair tiles)
    auto produce = [&](auto& cur, const CUtensorMap* map, const ConvGeom& g, uint8_t* base, int stage_bytes,
                       bool is_a) {
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = unit; tile < num_tiles; tile += units) {
            const int mn = tile % num_mn, split = tile / num_mn;
            const int o = is_a ? (mn % num_m) * TM + static_cast<int>(rank) * kBM
                               : (mn / num_m) * BN + static_cast<int>(rank) * C::kBNc;
            const int kb0 = split * sk.kps;
            const int kb_end = min(nk, (split + 1) * sk.kps);
            cur.init(g, o, kb0);
            for (int kb = kb0; kb < kb_end; ++kb) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                Tma<CG> t;
                t.bar = &full_bar[stage];
                t.bar_c = 0;
                if (CG == 1) {
                    mbar_arrive_expect_tx(&full_bar[stage], stage_bytes);
                } else {
                    // both CTAs' bytes land on the leader's full barrier
                    t.bar_c = mapa_shared(smem_u32(&full_bar[stage]), 0);
                    if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * stage_bytes);
                }
                cur.load(t, map, g, base + stage * stage_bytes, o);
                cur.advance(g);
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    };
    // row-reuse producers (no split-K): stage j of a tile = (column tap s,
    // channel block cb), s outer; A box rows [h0 + off, h0 + off + bh + ksz - 1)
    auto produce_rr = [&](bool is_a) {
        int stage = 0;
        uint32_t phase = 0;
        const int nj = ga.ksz * ga.cblocks;
        const int tx = is_a ? stA : stB;
        for (int tile = unit; tile < num_tiles; tile += units) {
            const int mn = tile % num_mn;
            const int m0 = (mn % num_m) * TM + static_cast<int>(rank) * kBM;
            const int n0 = (mn / num_m) * BN + static_cast<int>(rank) * C::kBNc;
            const int img = m0 / ga.howo, h0 = (m0 - img * ga.howo) / ga.wo;
            int sc = 0, cb = 0;
            for (int j = 0; j < nj; ++j) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                Tma<CG> t;
                t.bar = &full_bar[stage];
                t.bar_c = 0;
                if (CG == 1) {
                    mbar_arrive_expect_tx(&full_bar[stage], tx);
                } else {
                    t.bar_c = mapa_shared(smem_u32(&full_bar[stage]), 0);
                    if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * tx);
                }
                if (is_a) {
                    t.d4(sA + stage * stA, &ta, cb * 32, sc + ga.off, h0 + ga.off, img);
                } else {
                    for (int r = 0; r < ga.ksz; ++r)
                        load_operand<B_MN, C::kBNc, CG>(t, &tb, gb, sB + stage * stB + r * C::kStageB, n0,
                                                        (r * ga.ksz + sc) * ga.cblocks + cb);
                }
                if (++cb == ga.cblocks) {
                    cb = 0;
                    ++sc;
                }
                if (++stage == nst) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    };
    if (warp == 0) {
        if (elect_one()) {
            if (ga.rr) {
                produce_rr(true);
            } else {
                OperandCursor<A_MN, kBM, CG> ca;
                produce(ca, &ta, ga, sA, C::kStageA, true);
            }
        }
        __syncwarp();
        griddep_launch_dependents();  // every load issued: release the stream successor
    } else if (warp == 3) {
        if (elect_one()) {
            if (ga.rr) {
                produce_rr(false);
            } else {
                OperandCursor<B_MN, C::kBNc, CG> cb;
                produce(cb, &tb, gb, sB, C::kStageB, false);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        // The whole issue loop runs on ONE elected thread with the operand
        // descriptors built once and advanced by adding to their start-address
        // field (desc_advance): re-deriving 8 descriptors per K block and
        // re-electing per block cost ~75 issue slots per 4 MMAs, more than
        // the 4 x 58 tensor cycles of an N = 64 pair block.
        if (leader && elect_one()) {
            constexpr uint32_t idesc = idesc_tf32(BN, A_MN, B_MN, TM);
            // K-major (SW128): the K8 step advances 32 B inside the 128 B swizzle
            // atom; 8-row groups 1 KB apart (SBO).  MN-major (SW128_BASE32B):
            // the K8 step advances 8 K rows (1 KB); 4-row K groups 512 B apart
            // (SBO), 32-wide MN atoms 4 KB apart (LBO).
            const uint64_t a0 = A_MN ? umma_desc<kLayoutSW128Base32>(smem_u32(sA), 4096, 512)
                                     : umma_desc<kLayoutSW128>(smem_u32(sA), 16, 1024);
            const uint64_t b0 = B_MN ? umma_desc<kLayoutSW128Base32>(smem_u32(sB), 4096, 512)
                                     : umma_desc<kLayoutSW128>(smem_u32(sB), 16, 1024);
            constexpr uint32_t a_kk = A_MN ? 1024 : 32, b_kk = B_MN ? 1024 : 32;
            const bool no_mma = (epi.dbg & 8) != 0;  // timing probe (DEV builds only)
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int tile = unit; tile < num_tiles; tile += units, ++local) {
                const int acc = local % C::kAcc;
                const uint32_t acc_phase = (local / C::kAcc) & 1;
                mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                const int split = tile / num_mn;
                const int kb0 = ga.rr ? 0 : split * sk.kps;
                const int kb_end = ga.rr ? ga.ksz * ga.cblocks : min(nk, (split + 1) * sk.kps);
                for (int kb = kb0; kb < kb_end; ++kb) {
                    mbar_wait(&full_bar[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = desc_advance(a0, stage * stA);
                    const uint64_t bd = desc_advance(b0, stage * stB);
                    if (ga.rr && !no_mma) {
                        // row tap r: the box rows shifted by r image rows (r * bw * 128 B)
                        for (int r = 0; r < ga.ksz; ++r) {
                            const uint64_t ar = desc_advance(ad, r * ga.bw * 128);
                            const uint64_t br = desc_advance(bd, r * C::kStageB);
#pragma unroll
                            for (int kk = 0; kk < kBK / 8; ++kk) {
                                const uint32_t accum = (kb != 0 || r != 0 || kk != 0) ? 1u : 0u;
                                if (CG == 2)
                                    mma_tf32_pair(d_tmem, desc_advance(ar, kk * a_kk), desc_advance(br, kk * b_kk),
                                                  idesc, accum);
                                else
                                    mma_tf32(d_tmem, desc_advance(ar, kk * a_kk), desc_advance(br, kk * b_kk), idesc,
                                             accum);
                            }
                        }
                    } else if (!no_mma) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint32_t accum = (kb != kb0 || kk != 0) ? 1u : 0u;
                            if (CG == 2)
                                mma_tf32_pair(d_tmem, desc_advance(ad, kk * a_kk), desc_advance(bd, kk * b_kk), idesc,
                                              accum);
                            else
                                mma_tf32(d_tmem, desc_advance(ad, kk * a_kk), desc_advance(bd, kk * b_kk), idesc,
                                         accum);
                        }
                    }
                    if (CG == 2) mma_commit_pair(&empty_bar[stage]);
                    else mma_commit(&empty_bar[stage]);
                    if (++stage == nst) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (CG == 2) mma_commit_pair(&tfull_bar[acc]);
                else mma_commit(&tfull_bar[acc]);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int q = warp & 3;              // TMEM lane quarter this warp may access
        const int half = (warp - 4) >> 2;    // 0 / 1: even / odd 32-column chunks (or alternate tiles)
        const int lane = threadIdx.x & 31;
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty_bar[0]), 0) : 0;
        const bool db = epi.db_partial != nullptr;
        const int ldb = (N + 31) & ~31;
        // one bias-gradient row per warp: with by-tile epilogues both warps of
        // a lane quarter accumulate EVERY column (of different tiles), so a
        // shared row was a read-modify-write race (intermittent db errors)
        float* db_row = db_s + (q * 2 + half) * ldb;
        if (db) {
            for (int i = lane; i < ldb; i += 32) db_row[i] = 0.f;
            epi_bar_sync();
        }
        // >= 2 tiles per CTA: the two warp groups take alternate tiles (two
        // tiles' epilogues in flight, each on its own TMEM accumulator);
        // otherwise they split the tile's column chunks
        uint64_t* mbar = epi_mask_bar(stg, warp - 4);
        uint32_t mphase = 0;
        if (ts.n && ts.mask) {
            if (lane == 0) {
                mbar_init(mbar, 1);
                fence_mbar_init();
            }
            __syncwarp();
        }
        if (sj.on)  // a previous GEMM's split-K reduction, under this GEMM's mainloop
            run_side_job(sj, static_cast<long long>(blockIdx.x) * (kEpiWarps * 32) + (threadIdx.x - 128),
                         static_cast<long long>(gridDim.x) * (kEpiWarps * 32), lane);
        const bool by_tile = num_tiles >= 2 * units;
        const int c_first = by_tile ? 0 : half, c_step = by_tile ? 1 : 2;
        int bsel = 0;  // staging box of the next store (alternates when ts.dbuf)
        int local = 0;
        for (int tile = unit; tile < num_tiles; tile += units, ++local) {
            if (by_tile && (local & 1) != half) continue;
            const int mn = tile % num_mn, split = tile / num_mn;
            const int m0 = (mn % num_m) * TM + static_cast<int>(rank) * kBM;
            const int n0 = (mn / num_m) * BN;
            const int acc = local % C::kAcc;
            const uint32_t acc_phase = (local / C::kAcc) & 1;
            // masked epilogues: the first chunk's ReLU-mask box is loaded while
            // the tile's MMAs run (its latency was exposed once per tile)
            const bool masked = ts.n && ts.mask && !(sk.splits > 1 || sk.partial) && !(epi.dbg & 4);
            const bool pf = masked && ts.mask_pf;
            if (pf && c_first < BN / 32)
                tma_mask_issue(ts, stg + (warp - 4) * 4096, mbar, lane, m0 + q * 32, n0 + c_first * 32, ts.pool2 != 0);
            mbar_wait(&tfull_bar[acc], acc_phase);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
#pragma unroll 1
            for (int c = c_first; c < ((epi.dbg & 4) ? 0 : BN / 32); c += c_step) {  // dbg 4: timing probe, no epilogue
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, r);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
                if (sk.splits > 1 || sk.partial) {  // raw partial sums for splitk_epilogue_kernel
                    const int nn = n0 + c * 32;
                    if (ts.n) {
                        if (!(epi.dbg & 2)) tma_store_partial(ts, epi_box(stg, warp - 4, bsel), lane, v, m0 + q * 32, nn, split);
                        bsel ^= ts.dbuf;
                    } else if (sk.trans) {  // [n][m]: for each column the warp's lanes write consecutive m
                        float* col = sk.ws + split * sk.stride + m;
                        if (m < M) {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (nn + i < N) col[static_cast<long long>(nn + i) * sk.ld] = v[i];
                        }
                    } else if (m < M && nn < N) {
                        store_row32(sk.ws + split * sk.stride + static_cast<long long>(m) * sk.ld, nn,
                                    N - nn < 32 ? N - nn : 32, v);
                    }
                } else {
                    if (ts.n && ts.pool2) {
                        uint8_t* buf = stg + (warp - 4) * 4096;
                        if (ts.mask) {
                            if (c != c_first || !pf) tma_mask_issue(ts, buf, mbar, lane, m0 + q * 32, n0 + c * 32, true);
                            tma_mask_apply_issued(buf, mbar, mphase, lane, v);
                        }
                        uint32_t code[8];
                        const unsigned char* ap =
                            epi.mg_argmax + static_cast<long long>(m < M ? m : 0) * epi.mg_uch + n0 + c * 32;
#pragma unroll
                        for (int i = 0; i < 8; ++i) code[i] = m < M ? __ldg(reinterpret_cast<const uint32_t*>(ap) + i) : 0u;
                        tma_merge_pool2_chunk(ts, buf, lane, v, code, m0 + q * 32, n0 + c * 32);
                    } else if (ts.n && ts.mask) {
                        if (c != c_first || !pf) tma_mask_issue(ts, stg + (warp - 4) * 4096, mbar, lane, m0 + q * 32, n0 + c * 32);
                        if (ts.res) {  // residual forward: conv + bias here, shortcut + ReLU from the box
                            epi_values32(epi, m, n0 + c * 32, v, lane, true);
                            tma_store_res_issued(ts, stg + (warp - 4) * 4096, mbar, mphase, lane, v, m0 + q * 32,
                                                 n0 + c * 32, epi.relu);
                        } else {
                            if (epi.mg_sg != nullptr && m < M) epi_merge_sg32(epi, m, n0 + c * 32, v);  // shortcut gradient
                            tma_store_masked_issued(ts, stg + (warp - 4) * 4096, mbar, mphase, lane, v, m0 + q * 32,
                                                    n0 + c * 32);
                        }
                    } else if (ts.n && epi.pl_on == 3) {
                        // 2x2 pool across the warp pair holding image rows 2y, 2y+1
                        // (pre-pool rows are not stored: nothing reads them)
                        epi_values32(epi, m, n0 + c * 32, v, lane);
                        stage_chunk(stg + (warp - 4) * 4096, lane, v);
                        pair_bar_sync(warp - 4);
                        const int pw = (warp - 4) & ~1;
                        epi_pool_pair(epi, m0 + (q & ~1) * 32, n0 + c * 32, lane, smem_u32(stg + pw * 4096),
                                      smem_u32(stg + (pw + 1) * 4096), q & 1);
                        pair_bar_sync(warp - 4);
                    } else if (ts.n) {
                        epi_values32(epi, m, n0 + c * 32, v, lane);
                        if (!(epi.dbg & 2)) tma_store_chunk(ts, epi_box(stg, warp - 4, bsel), lane, v, m0 + q * 32, n0 + c * 32);
                        bsel ^= ts.dbuf;
                        if (epi.pl_on == 2) {  // window partners from the staging box just written
                            __syncwarp();
                            epi_pool32_smem(epi, m, n0 + c * 32, v, lane, smem_u32(stg + (warp - 4) * 4096));
                            __syncwarp();
                        } else if (epi.pl_on) {
                            epi_pool32(epi, m, n0 + c * 32, v, lane);
                        }
                    } else if (!(epi.dbg & 2)) {
                        epilogue32(epi, m, n0 + c * 32, v);
                        if (epi.pl_on) epi_pool32(epi, m, n0 + c * 32, v, lane);
                    }
                    if (db && n0 + c * 32 < N) {
                        if (m >= M) {
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] = 0.f;
                        }
                        db_accumulate(db_row, n0 + c * 32, N, v, lane);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                const uint32_t cnt = by_tile ? 2u : 1u;  // by_tile: 4 warps stand for all 8
                if (CG == 2) mbar_arrive_remote_n(tempty_leader + acc * sizeof(uint64_t), cnt);
                else mbar_arrive_n(&tempty_bar[acc], cnt);
            }
            if (sk.splits > 1 && sk.fixup && !(epi.dbg & 6)) {
                // publish this warp's partial chunks; the last writer of the slot reduces
                if (ts.n && lane == 0) bulk_wait<0>();
                fence_proxy_async_global();
                __threadfence();
                __syncwarp();
                const int slot = by_tile ? q : q * 2 + half;
                int* ctr = sk.counters + (static_cast<long long>(mn) * CG + rank) * 8 + slot;
                int old = 0;
                if (lane == 0) old = atomicAdd(ctr, 1);
                old = __shfl_sync(0xffffffffu, old, 0);
                if (old == sk.splits - 1) {
                    __threadfence();
#pragma unroll 1
                    for (int c = c_first; c < BN / 32; c += c_step) {
                        const int nn = n0 + c * 32;
                        if (nn >= N) break;
                        const int nv = N - nn < 32 ? N - nn : 32;
                        float v[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0.f;
                        if (m < M) {
#pragma unroll 1
                            for (int sp = 0; sp < sk.splits; ++sp) {
                                if (sk.trans) {
                                    const float* col = sk.ws + sp * sk.stride + m;
#pragma unroll
                                    for (int i = 0; i < 32; ++i)
                                        if (i < nv) v[i] += __ldcg(col + static_cast<long long>(nn + i) * sk.ld);
                                } else {
                                    const float* row = sk.ws + sp * sk.stride + static_cast<long long>(m) * sk.ld + nn;
                                    if (nv == 32 && (sk.ld & 3) == 0) {
#pragma unroll
                                        for (int i = 0; i < 32; i += 4) {
                                            const float4 t = __ldcg(reinterpret_cast<const float4*>(row + i));
                                            v[i] += t.x;
                                            v[i + 1] += t.y;
                                            v[i + 2] += t.z;
                                            v[i + 3] += t.w;
                                        }
                                    } else {
#pragma unroll
                                        for (int i = 0; i < 32; ++i)
                                            if (i < nv) v[i] += __ldcg(row + i);
                                    }
                                }
                            }
                        }
                        epilogue32(epi, m, nn, v);
                    }
                    if (lane == 0) *ctr = 0;  // re-armed for the next launch
                }
            }
        }
        if (db) {  // the quarter's two rows, in a fixed order
            epi_bar_sync();
            if (half == 0) {
                float* out = epi.db_partial + (static_cast<long long>(blockIdx.x) * 4 + q) * N;
                for (int i = lane; i < N; i += 32) out[i] = db_row[i] + db_row[ldb + i];
            }
        }
        if (ts.n && lane == 0) bulk_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem_base, C::kTmemCols);
        else tmem_dealloc(tmem_base, C::kTmemCols);
    }
}

// Split-K reduction + the GEMM's real epilogue.  The workspace is [m][n]
// (pitch sk.ld), or [n][m] when sk.trans (the dW^T SGD epilogue, whose W[n][m]
// writes coalesce along m).  Work item = one workspace row x 4 consecutive
// columns.  PHASES = 1: a thread sums every split of its item in order.
// PHASES = 8 (many splits, e.g. the 148-way wgrad of VGG conv1): phase y sums
// splits y, y+8, ... in order, then phase 0 adds the 8 phase sums in order
// (a fixed tree: deterministic).
template <int PHASES>
__global__ void __launch_bounds__(256) splitk_epilogue_kernel(
    const __grid_constant__ EpiParams epi, const __grid_constant__ SplitK sk, int M, int N) {
    constexpr int kItems = 256 / PHASES;
    __shared__ float4 part[PHASES][kItems];
    griddep_wait();  // launched programmatically after its GEMM
    const int bblocks = sk.bias != nullptr ? (sk.bu + 31) / 32 : 0;
    if (static_cast<int>(blockIdx.x) >= static_cast<int>(gridDim.x) - bblocks) {
        // bias job: column = t % 32, phase y = t / 32 sums chunks y, y+8, ...
        // in order; phase sums added in order 0..7 (deterministic)
        __shared__ float bsh[8][33];
        const int t = threadIdx.y * blockDim.x + threadIdx.x;
        const int col = (blockIdx.x - (gridDim.x - bblocks)) * 32 + (t & 31), y = t >> 5;
        const float acc = col < sk.bu ? bias_chunk_sum(sk.bpart, sk.bu, col, y, sk.bchunks) : 0.f;
        bsh[y][t & 31] = acc;
        __syncthreads();
        if (y == 0 && col < sk.bu) {
            float g = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) g += bsh[j][t & 31];
            sk.bias[col] -= static_cast<float>(*epi.alpha) * (g * epi.inv_b);
        }
        return;
    }
    const int R = sk.trans ? N : M;
    const int Cc = sk.trans ? M : N;
    const int cq = (Cc + 3) / 4;
    const long long item = static_cast<long long>(blockIdx.x) * kItems + threadIdx.x;
    const bool live = item < static_cast<long long>(R) * cq;
    const int r = live ? static_cast<int>(item / cq) : 0;
    const int c4 = live ? static_cast<int>(item - static_cast<long long>(r) * cq) * 4 : 0;
    const int nc = Cc - c4 < 4 ? Cc - c4 : 4;
    const bool vec = nc == 4 && (sk.ld & 3) == 0;
    const long long off = static_cast<long long>(r) * sk.ld + c4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
#pragma unroll 4
        for (int sp = threadIdx.y; sp < sk.splits; sp += PHASES) {
            const float* src = sk.ws + static_cast<long long>(sp) * sk.stride + off;
            float4 t;
            if (vec) {
                t = __ldcg(reinterpret_cast<const float4*>(src));
            } else {
                t.x = __ldcg(src);
                t.y = nc > 1 ? __ldcg(src + 1) : 0.f;
                t.z = nc > 2 ? __ldcg(src + 2) : 0.f;
                t.w = nc > 3 ? __ldcg(src + 3) : 0.f;
            }
            acc.x += t.x;
            acc.y += t.y;
            acc.z += t.z;
            acc.w += t.w;
        }
    }
    float a[4] = {acc.x, acc.y, acc.z, acc.w};
    if (PHASES > 1) {
        part[threadIdx.y][threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.y != 0) return;
        a[0] = a[1] = a[2] = a[3] = 0.f;
#pragma unroll
        for (int y = 0; y < PHASES; ++y) {
            const float4 t = part[y][threadIdx.x];
            a[0] += t.x;
            a[1] += t.y;
            a[2] += t.z;
            a[3] += t.w;
        }
    }
    if (!live) return;
    if (sk.trans) {  // EPI_SGD on dW^T: row r = n, columns = m
        const float alpha = static_cast<float>(*epi.alpha);
        float* w = epi.W + static_cast<long long>(r) * epi.ldw + c4;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j < nc) {
                const float g = a[j] * epi.inv_b;
                bad |= !isfinite(g);
                w[j] -= alpha * g;
            }
        }
        if (bad && epi.flag != nullptr) atomicOr(epi.flag, 1);
        return;
    }
    const long long row_off = epi.mode == EPI_STORE ? epi_store_row(epi, r) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < nc) epilogue1(epi, r, c4 + j, a[j], row_off);
}


// The split-K reduction + epilogue of a GEMM (p.sk.splits partial slices at
// p.sk.ws, summed in slice order) as its own launch.
cudaError_t launch_splitk_reduce(const TcGemmPlan& p, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    const long long R = p.sk.trans ? p.N : p.M, Cc = p.sk.trans ? p.M : p.N;
    const long long items = R * ((Cc + 3) / 4);
    const unsigned bblocks = p.sk.bias != nullptr ? static_cast<unsigned>((p.sk.bu + 31) / 32) : 0u;
    cudaLaunchConfig_t rc{};
    rc.stream = s;
    cudaLaunchAttribute ra[1];
    ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ra[0].val.programmaticStreamSerializationAllowed = 1;
    rc.attrs = ra;
    rc.numAttrs = pdl_enabled() ? 1 : 0;
    if (p.sk.splits >= 64) {  // e.g. conv1's 148-way wgrad: 8 items x 32 phases per block
        rc.gridDim = dim3(static_cast<unsigned>((items + 7) / 8) + bblocks);
        rc.blockDim = dim3(8, 32);
        e = cudaLaunchKernelEx(&rc, splitk_epilogue_kernel<32>, p.epi, p.sk, p.M, p.N);
    } else if (p.sk.splits >= 16) {
        rc.gridDim = dim3(static_cast<unsigned>((items + 31) / 32) + bblocks);
        rc.blockDim = dim3(32, 8);
        e = cudaLaunchKernelEx(&rc, splitk_epilogue_kernel<8>, p.epi, p.sk, p.M, p.N);
    } else {
        rc.gridDim = dim3(static_cast<unsigned>((items + 255) / 256) + bblocks);
        rc.blockDim = dim3(256, 1);
        e = cudaLaunchKernelEx(&rc, splitk_epilogue_kernel<1>, p.epi, p.sk, p.M, p.N);
    }

    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <bool A_MN, bool B_MN, int BN, int CG>
cudaError_t launch_t(const TcGemmPlan& p, cudaStream_t s) {
    using C = TcCfg<BN, CG>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 1024 + p.stages * (p.stage_bytes ? p.stage_bytes : C::kStageBytes) + 256 + p.db_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<A_MN, B_MN, BN, CG>, p.ta, p.tb, p.M, p.N, p.K, p.epi,
                                       p.ga, p.gb, p.sk, p.ts, p.stages, p.sj);
    const bool probe_no_reduce = dev_knob("PPB_PROBE_NO_REDUCE");  // timing probe (wrong results)
    if (e != cudaSuccess || p.sk.splits <= 1 || p.sk.fixup || p.sk.deferred || p.sk.partial || probe_no_reduce)
        return e;
    return launch_splitk_reduce(p, s);
}

}  // namespace

}  // namespace ppb
