// Halo-reuse implicit-GEMM 3x3 convolution for sm_100a (tcgen05, TF32).
//
// The rank-4 implicit GEMM in gemm_tc.cu stages a fresh 128-pixel x 32-channel
// A box for every one of the 9 taps, so A crosses L2 -> SM nine times.  On the
// narrow layers (C_out <= 128, large spatial grids) that traffic, not the
// tensor core, sets the speed: ~42 B/clk/SM of TMA service against a 128 x 64
// x 32 MMA block that needs ~130 clk.
//
// Here the GEMM rows are positions of the PADDED grid [imgs][hp][wp] (the
// rows at pad positions are computed and dropped by the epilogue, ~13% extra
// MMA work at 32x32, ~27% at 16x16).  In that space tap (r, s) is a constant
// row shift r*wp + s, so one TMA box of 128 + 2*(wp+1) consecutive rows (the
// "halo") per 32-channel block serves all 9 taps: the MMA issuer points the
// SW128 K-major A descriptor at halo row r*wp + s (rows are 128 B apart, the
// swizzle phase follows the absolute smem address exactly as the TMA wrote it).
// A traffic drops ~6x.  B (the weights) is then the larger stream: when the
// CTA's whole B column slice (BN/CG rows x 9*C) fits beside two halo stages it
// is loaded ONCE per CTA and stays resident (VGG conv2 / conv3 and their dgrads);
// otherwise it streams through its own ring.
//
//   warp 0      TMA producer: halo ring (2-4 stages)
//   warp 3      TMA producer: resident B slice (once) or the B ring
//   warp 1      MMA issuer (leader CTA; CG = 2 -> M = 256 over a CTA pair)
//   warp 2      TMEM allocator (2 x BN accumulator columns)
//   warps 4..7  epilogue: padded position -> output pixel (or skip) -> the
//               shared epilogue32 (bias/ReLU/remap/slots/mask)
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "dev_knobs.h"
#include "epilogue.cuh"
#include "gemm_tc.h"
#include "ptx.cuh"
#include "tc_common.cuh"

namespace ppb {

namespace {

std::atomic<unsigned> g_halo_attr{0};

constexpr int kHaloThreads = 128 + 32 * kEpiWarps;
constexpr int kHaloMaxRows = 256;  // TMA box limit
constexpr int kHaloSmemMax = 227 * 1024;
constexpr int kHaloReserve = 1024 + 1024;  // alignment slack + barriers

template <int BN, int CG>
struct HaloCfg {
    static constexpr int kBNc = BN / CG;
    static constexpr int kStageB = kBNc * kBK * 4;
    // accumulator ring: 4 deep up to BN = 128 (the epilogue of a narrow tile
    // can lag the MMAs by more than one tile), 2 at BN = 256 (512 columns)
    static constexpr int kAcc = BN <= 128 ? 4 : 2;
    static constexpr int kTmemCols = kAcc * BN;
};

template <bool B_MN, int BN, int CG>
__global__ void __launch_bounds__(kHaloThreads, 1)
    halo_conv_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int N,
                     const __grid_constant__ HaloGeom hg, const __grid_constant__ EpiParams epi,
                     const __grid_constant__ ConvGeom gb, const __grid_constant__ TmaStore ts) {
    using C = HaloCfg<BN, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    const int kHaloStages = hg.hstages, kHaloStageBytes = hg.hstage_bytes;
    const int kBStages = hg.bstages;  // resident: one slot per K block, loaded once
    uint8_t* sH = smem;
    uint8_t* sB = smem + kHaloStages * kHaloStageBytes;
    uint64_t* hfull = reinterpret_cast<uint64_t*>(sB + kBStages * C::kStageB);
    uint64_t* hempty = hfull + kHaloStages;
    uint64_t* bfull = hempty + kHaloStages;
    uint64_t* bempty = bfull + kBStages;
    uint64_t* tfull = bempty + kBStages;  // [kAcc]
    uint64_t* tempty = tfull + C::kAcc;    // [kAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::kAcc);
    float* db_s = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(hfull) + 1024);  // [4][ldb] (EPI_MERGE db)
    uint8_t* stg = reinterpret_cast<uint8_t*>(hfull) + ts.stage_off;                    // TMA-store staging

    const int warp = threadIdx.x / 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    constexpr int TM = kBM * CG;
    const int num_m = static_cast<int>((hg.Mp + TM - 1) / TM);
    const int num_n = (N + BN - 1) / BN;
    const int num_tiles = num_m * num_n;
    const int unit = blockIdx.x / CG;
    const int units = gridDim.x / CG;
    const int cblocks = hg.cblocks;
    const uint32_t halo_bytes = static_cast<uint32_t>(hg.rows) * 128u;

    if (warp == 0 && elect_one()) {
        tma_prefetch(&ta);
        tma_prefetch(&tb);
        for (int s = 0; s < kHaloStages; ++s) {
            mbar_init(&hfull[s], 1);
            mbar_init(&hempty[s], 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        for (int i = 0; i < C::kAcc; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps * CG);
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

    if (warp == 0) {
        // ------------------------------------------------ TMA producer: halo boxes
        if (elect_one()) {
            int hs = 0;
            uint32_t hph = 0;
            for (int tile = unit; tile < num_tiles; tile += units) {
                const long long p0 = static_cast<long long>(tile % num_m) * TM + static_cast<long long>(rank) * kBM;
                for (int cb = 0; cb < cblocks; ++cb) {
                    mbar_wait(&hempty[hs], hph ^ 1);
                    Tma<CG> th;
                    th.bar = &hfull[hs];
                    th.bar_c = 0;
                    if (CG == 1) {
                        mbar_arrive_expect_tx(&hfull[hs], halo_bytes);
                    } else {
                        th.bar_c = mapa_shared(smem_u32(&hfull[hs]), 0);
                        if (leader) mbar_arrive_expect_tx(&hfull[hs], 2 * halo_bytes);
                    }
                    // rows [p0 - wp - 1, p0 + 128 + wp + 1): out-of-range rows are zero-filled
                    th.d2(sH + hs * kHaloStageBytes, &ta, cb * 32, static_cast<int>(p0 - hg.wp - 1));
                    if (++hs == kHaloStages) {
                        hs = 0;
                        hph ^= 1;
                    }
                }
            }
        }
        __syncwarp();
        griddep_launch_dependents();  // every halo load issued: release the stream successor
    } else if (warp == 3) {
        // ------------------------------------------------ TMA producer: B (weights)
        if (elect_one()) {
            auto issue = [&](int slot, int n0, int kb) {
                Tma<CG> t;
                t.bar = &bfull[slot];
                t.bar_c = 0;
                if (CG == 1) {
                    mbar_arrive_expect_tx(&bfull[slot], C::kStageB);
                } else {
                    t.bar_c = mapa_shared(smem_u32(&bfull[slot]), 0);
                    if (leader) mbar_arrive_expect_tx(&bfull[slot], 2 * C::kStageB);
                }
                load_operand<B_MN, C::kBNc, CG>(t, &tb, gb, sB + slot * C::kStageB, n0, kb);
            };
            if (hg.resident) {
                // the whole B slice of this CTA (one column tile), once: every K
                // block on its own barrier so the first MMAs start early
                for (int kb = 0; kb < 9 * cblocks; ++kb) issue(kb, static_cast<int>(rank) * C::kBNc, kb);
            } else {
                int bs = 0;
                uint32_t bph = 0;
                for (int tile = unit; tile < num_tiles; tile += units) {
                    const int n0 = (tile / num_m) * BN + static_cast<int>(rank) * C::kBNc;
                    for (int cb = 0; cb < cblocks; ++cb) {
                        for (int tap = 0; tap < 9; ++tap) {
                            mbar_wait(&bempty[bs], bph ^ 1);
                            issue(bs, n0, tap * cblocks + cb);
                            if (++bs == kBStages) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        // One elected thread runs the whole issue loop; descriptors are built
        // once and advanced by address adds (desc_advance).  Per tap the issue
        // cost was ~124 instructions (descriptor re-derivation, re-election)
        // against 4 x 58 tensor cycles at N = 64: the kernel was issue-bound
        // (ncu source page: the MMA warp never waited, the epilogue and the
        // halo producer waited on it).
        if (leader && elect_one()) {
            constexpr uint32_t idesc = idesc_tf32(BN, false, B_MN, TM);
            constexpr uint32_t b_kk = B_MN ? 1024 : 32;
            const uint64_t h0 = umma_desc<kLayoutSW128>(smem_u32(sH), 16, 1024);
            const uint64_t b0 = B_MN ? umma_desc<kLayoutSW128Base32>(smem_u32(sB), 4096, 512)
                                     : umma_desc<kLayoutSW128>(smem_u32(sB), 16, 1024);
            uint32_t roff[9];  // tap (r, s) = halo row shift r * wp + s, in bytes
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
                int ro = (tap / 3) * hg.wp + tap % 3;
                if (hg.dbg & 1) ro &= ~7;  // timing probe only (wrong results)
                roff[tap] = static_cast<uint32_t>(ro) * 128u;
            }
            const bool no_mma = (hg.dbg & 8) != 0;  // timing probe (DEV builds only)
            int hs = 0, bs = 0;
            uint32_t hph = 0, bph = 0;
            int local = 0;
            for (int tile = unit; tile < num_tiles; tile += units, ++local) {
                const int acc = local % C::kAcc;
                const uint32_t acc_phase = (local / C::kAcc) & 1;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int cb = 0; cb < cblocks; ++cb) {
                    if (!(hg.dbg & 4) || local == 0) mbar_wait(&hfull[hs], hph);
                    const uint64_t hd = desc_advance(h0, hs * kHaloStageBytes);
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap) {
                        const int kb = tap * cblocks + cb;
                        if (hg.resident) {
                            if (local == 0) mbar_wait(&bfull[kb], 0);
                        } else {
                            mbar_wait(&bfull[bs], bph);
                        }
                        tc_fence_after();
                        const uint64_t ad = desc_advance(hd, roff[tap]);
                        const uint64_t bd = desc_advance(b0, (hg.resident ? kb : bs) * C::kStageB);
                        if (!no_mma) {
#pragma unroll
                            for (int kk = 0; kk < kBK / 8; ++kk) {
                                const uint32_t accum = (cb != 0 || tap != 0 || kk != 0) ? 1u : 0u;
                                if (CG == 2)
                                    mma_tf32_pair(d_tmem, desc_advance(ad, kk * 32), desc_advance(bd, kk * b_kk),
                                                  idesc, accum);
                                else
                                    mma_tf32(d_tmem, desc_advance(ad, kk * 32), desc_advance(bd, kk * b_kk), idesc,
                                             accum);
                            }
                        }
                        if (!hg.resident) {
                            if (CG == 2) mma_commit_pair(&bempty[bs]);
                            else mma_commit(&bempty[bs]);
                            if (++bs == kBStages) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                    if (CG == 2) mma_commit_pair(&hempty[hs]);
                    else mma_commit(&hempty[hs]);
                    if (++hs == kHaloStages) {
                        hs = 0;
                        hph ^= 1;
                    }
                }
                if (CG == 2) mma_commit_pair(&tfull[acc]);
                else mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int q = warp & 3;              // TMEM lane quarter this warp may access
        const int half = (warp - 4) >> 2;    // 0 / 1: even / odd 32-column chunks
        const int lane = threadIdx.x & 31;
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0;
        const int hpwp = hg.hp * hg.wp;
        uint64_t* mbar = epi_mask_bar(stg, warp - 4);
        uint32_t mphase = 0;
        if (ts.n && ts.mask) {
            if (lane == 0) {
                mbar_init(mbar, 1);
                fence_mbar_init();
            }
            __syncwarp();
        }
        const bool db = epi.db_partial != nullptr;
        const int ldb = (N + 31) & ~31;
        float* db_row = db_s + q * ldb;
        if (db) {
            if (half == 0)
                for (int i = lane; i < ldb; i += 32) db_row[i] = 0.f;
            epi_bar_sync();
        }
        int local = 0;
        int msel = 0;  // staging box of the next masked chunk (alternates with ts.dbuf)
        const bool masked = ts.n && ts.mask;
        // two staging boxes per warp: the mask box of this warp's NEXT chunk
        // (the next tile's first chunk after the last) is loaded as soon as the
        // current chunk's store is issued, so its latency hides behind a whole
        // chunk of epilogue work, not only behind the tile's MMAs
        // shortcut-gradient merge: the second box holds the shortcut rows, so no
        // look-ahead mask load (box 0 only, both boxes loaded per chunk)
        const bool sgbox = masked && ts.sg && ts.dbuf;
        const bool ahead = masked && ts.mask_pf && ts.dbuf && !sgbox;
        auto mask_issue = [&](int t, int c) {
            const long long pp = static_cast<long long>(t % num_m) * TM + static_cast<long long>(rank) * kBM;
            tma_mask_issue(ts, epi_box(stg, warp - 4, msel), mbar, lane, static_cast<int>(pp) + q * 32,
                           (t / num_m) * BN + c * 32, false, ts.dbuf);
        };
        if (ahead && unit < num_tiles && half < BN / 32) mask_issue(unit, half);
        for (int tile = unit; tile < num_tiles; tile += units, ++local) {
            const long long p0 = static_cast<long long>(tile % num_m) * TM + static_cast<long long>(rank) * kBM;
            const int n0 = (tile / num_m) * BN;
            const int acc = local % C::kAcc;
            const uint32_t acc_phase = (local / C::kAcc) & 1;
            // padded position -> output pixel, -1 on the pad ring / past the end
            const long long pos = p0 + q * 32 + lane;
            int m = -1;
            if (pos < hg.Mp) {
                const int img = static_cast<int>(pos / hpwp);
                const int rem = static_cast<int>(pos - static_cast<long long>(img) * hpwp);
                const int hh = rem / hg.wp, ww = rem - hh * hg.wp;
                if (hh >= 1 && hh <= hg.ho && ww >= 1 && ww <= hg.wo) m = (img * hg.ho + hh - 1) * hg.wo + ww - 1;
            }
            // the first chunk's ReLU-mask box is loaded while the tile's MMAs run
            // (with two staging boxes per warp, while the previous chunk's store
            // still reads the other box)
            if (masked && ts.mask_pf && !ahead && half < BN / 32) {
                if (sgbox)
                    tma_mask_sg_issue(ts, epi_box(stg, warp - 4, 0), epi_box(stg, warp - 4, 1), mbar, lane,
                                      static_cast<int>(p0) + q * 32, n0 + half * 32);
                else
                    tma_mask_issue(ts, epi_box(stg, warp - 4, msel), mbar, lane, static_cast<int>(p0) + q * 32,
                                   n0 + half * 32, false, ts.dbuf);
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = half; c < BN / 32; c += 2) {
                uint32_t rr[32];
                tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, rr);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = m >= 0 ? __uint_as_float(rr[i]) : 0.f;
                if (masked) {  // the mask is zero on the ring
                    uint8_t* box = epi_box(stg, warp - 4, msel);
                    if (sgbox) {
                        uint8_t* box1 = epi_box(stg, warp - 4, 1);
                        if (c != half || !ts.mask_pf)
                            tma_mask_sg_issue(ts, box, box1, mbar, lane, static_cast<int>(p0) + q * 32, n0 + c * 32);
                        tma_store_masked_sg_issued(ts, box, box1, mbar, mphase, lane, v, static_cast<int>(p0) + q * 32,
                                                   n0 + c * 32);
                    } else if (!ahead && (c != half || !ts.mask_pf)) {
                        tma_mask_issue(ts, box, mbar, lane, static_cast<int>(p0) + q * 32, n0 + c * 32, false,
                                       ts.dbuf);
                    }
                    if (sgbox) {
                        // stored above
                    } else if (ts.res) {  // residual forward: conv + bias here, shortcut + ReLU from the box
                        epi_values32(epi, m, n0 + c * 32, v, lane, true);
                        if (m < 0) {  // pad-ring rows keep the destination's zeros (the box's ring is zero)
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] = 0.f;
                        }
                        tma_store_res_issued(ts, box, mbar, mphase, lane, v, static_cast<int>(p0) + q * 32,
                                             n0 + c * 32, epi.relu);
                    } else {
                        if (epi.mg_sg != nullptr && m >= 0) epi_merge_sg32(epi, m, n0 + c * 32, v);  // shortcut gradient
                        tma_store_masked_issued(ts, box, mbar, mphase, lane, v, static_cast<int>(p0) + q * 32,
                                                n0 + c * 32);
                    }
                    if (!sgbox) msel ^= ts.dbuf;
                    if (ahead) {
                        if (c + 2 < BN / 32) mask_issue(tile, c + 2);
                        else if (tile + units < num_tiles) mask_issue(tile + units, half);
                    }
                } else if (ts.n) {  // pad-ring rows store zeros (the destination's own ring)
                    epi_values32(epi, m, n0 + c * 32, v, lane);
                    if (m < 0) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = 0.f;
                    }
                    if (!(hg.dbg & 2))
                        tma_store_chunk(ts, stg + (warp - 4) * 4096, lane, v, static_cast<int>(p0) + q * 32, n0 + c * 32);
                } else if (m >= 0 && !(hg.dbg & 2)) {
                    epilogue32(epi, m, n0 + c * 32, v);
                }
                if (db && n0 + c * 32 < N) db_accumulate(db_row, n0 + c * 32, N, v, lane);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_remote_n(tempty_leader + acc * sizeof(uint64_t), 1);
                else mbar_arrive(&tempty[acc]);
            }
        }
        if (db) {  // both warps of the quarter accumulated into db_row (disjoint columns)
            epi_bar_sync();
            if (half == 0) {
                float* out = epi.db_partial + (static_cast<long long>(blockIdx.x) * 4 + q) * N;
                for (int i = lane; i < N; i += 32) out[i] = db_row[i];
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

template <bool B_MN, int BN, int CG>
cudaError_t launch_halo_t(const TcGemmPlan& p, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    if ((g_halo_attr.load() & (1u << (dev & 31))) == 0) {
        cudaError_t e = halo_conv_init_device();
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(kHaloThreads);
    cfg.dynamicSmemBytes = p.hg.smem;
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
    return cudaLaunchKernelEx(&cfg, halo_conv_kernel<B_MN, BN, CG>, p.ta, p.tb, p.N, p.hg, p.epi, p.gb, p.ts);
}

template <bool B_MN>
cudaError_t launch_halo_bn(const TcGemmPlan& p, cudaStream_t s) {
    if (p.cg == 2) {
        switch (p.bn) {
            case 64: return launch_halo_t<B_MN, 64, 2>(p, s);
            case 128: return launch_halo_t<B_MN, 128, 2>(p, s);
            default: return launch_halo_t<B_MN, 256, 2>(p, s);
        }
    }
    switch (p.bn) {
        case 64: return launch_halo_t<B_MN, 64, 1>(p, s);
        case 128: return launch_halo_t<B_MN, 128, 1>(p, s);
        default: return launch_halo_t<B_MN, 256, 1>(p, s);
    }
}

}  // namespace

cudaError_t halo_conv_init_device() {
    cudaError_t e = cudaSuccess;
    auto set = [&](auto kernel, int smem) {
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    };
#define PPB_HSET(BM)                                                     \
    set(halo_conv_kernel<BM, 64, 1>, kHaloSmemMax);             \
    set(halo_conv_kernel<BM, 128, 1>, kHaloSmemMax);           \
    set(halo_conv_kernel<BM, 256, 1>, kHaloSmemMax);           \
    set(halo_conv_kernel<BM, 64, 2>, kHaloSmemMax);             \
    set(halo_conv_kernel<BM, 128, 2>, kHaloSmemMax);           \
    set(halo_conv_kernel<BM, 256, 2>, kHaloSmemMax);
    PPB_HSET(false)
    PPB_HSET(true)
#undef PPB_HSET
    int dev = 0;
    cudaGetDevice(&dev);
    if (e == cudaSuccess) g_halo_attr.fetch_or(1u << (dev & 31));
    return e;
}

// A conv forward / dgrad descriptor (conv.h) whose A operand is a 3x3 implicit
// conv over a padded grid with a one-pixel ring, whose output grid equals the
// padded grid's interior, and where the padded-space overhead is modest.
bool halo_conv_eligible(const GemmDesc& d) {
    const ConvGeom& g = d.a.geom;
    if (g.mode != OP_CONV_ROWS || d.a.mn_major || g.ksz != 3 || g.off != 0) return false;
    if (d.b.geom.mode != OP_DENSE && d.b.geom.mode != OP_WFLIP) return false;
    const int wo = g.wo, ho = g.howo / g.wo;
    if (d.a.wp != wo + 2 || d.a.hp != ho + 2) return false;
    if (d.a.wp + 1 > (kHaloMaxRows - kBM) / 2) return false;
    if (static_cast<long long>(d.a.imgs) * d.a.hp * d.a.wp >= (1LL << 31)) return false;
    if (d.M != d.a.imgs * ho * wo || d.K != 9 * g.cblocks * 32) return false;
    const double waste = static_cast<double>(d.a.hp) * d.a.wp / (static_cast<double>(ho) * wo);
    return waste <= 1.3;
}

// Automatic choice between the halo kernel and the rank-4 implicit GEMM for an
// eligible descriptor, measured with the TMA-store epilogues (VGG,
// profile_ops): a pooled backward merge needs the stride-2 quadrant boxes the
// padded-position tiles cannot form (conv3 dgrad 107.6 vs 91.1 us), and
// MN-major (flipped-weight) B at N >= 128 streams B beside the halo (conv4
// dgrad 113.7 vs 97.3 us).  Step 2.270 -> 2.244 ms.
bool halo_conv_preferred(const GemmDesc& d) {
    static const bool always = dev_knob("PPB_HALO_ALWAYS");
    if (always) return true;
    if (d.epi.mode == EPI_MERGE && d.epi.mg_pool == 2) return false;
    if (d.b.mn_major && d.N >= 128) return false;
    // pre-pool output rows (not a padded grid: the halo epilogue would fall back
    // to per-thread stores) at N <= 64: conv2 forward 158.7 vs 152.5 us
    static const bool u64 = !dev_knob("PPB_HALO_U64");
    if (u64 && d.epi.mode == EPI_STORE && !d.epi.remap && d.N <= 64) return false;
    return true;
}

// force: 0 = automatic tile choice; 1000 + bn = 1-CTA tiles of width bn;
// 2000 + bn = CTA-pair tiles (256 x bn).
bool halo_conv_prepare(const GemmDesc& d, TcGemmPlan* out, int force, char* err, size_t errlen) {
    if (!halo_conv_eligible(d)) {
        snprintf(err, errlen, "conv descriptor not eligible for the halo kernel");
        return false;
    }
    TcGemmPlan p;
    p.halo = 1;
    p.M = d.M;
    p.N = d.N;
    p.K = d.K;
    p.a_mn = false;
    p.b_mn = d.b.mn_major;
    p.epi = d.epi;
    p.epi.M = d.M;
    p.epi.N = d.N;
    p.ga = d.a.geom;
    p.gb = d.b.geom;
    HaloGeom& hg = p.hg;
    hg.wp = d.a.wp;
    hg.hp = d.a.hp;
    hg.wo = d.a.geom.wo;
    hg.ho = d.a.geom.howo / d.a.geom.wo;
    hg.cblocks = d.a.geom.cblocks;
    hg.rows = kBM + 2 * (hg.wp + 1);
    hg.Mp = static_cast<long long>(d.a.imgs) * hg.hp * hg.wp;
    hg.dbg = static_cast<int>(dev_knob_uint("PPB_HALO_DBG"));  // timing probes only
    int bn, cg;
    if (force >= 2000) {
        cg = 2;
        bn = force - 2000;
    } else if (force >= 1000) {
        cg = 1;
        bn = force - 1000;
    } else {
        // pairs halve the per-SM B bytes; pick the narrowest width covering N
        // (or 256-wide column tiles)
        cg = hg.Mp > 2 * kBM ? 2 : 1;
        bn = d.N <= 64 ? 64 : (d.N <= 128 ? 128 : 256);
    }
    if (bn != 64 && bn != 128 && bn != 256) {
        snprintf(err, errlen, "halo conv: unsupported tile width %d", bn);
        return false;
    }
    p.bn = bn;
    p.cg = cg;
    // shared-memory plan: halo ring + either the whole B column slice resident
    // (one column tile, fits next to >= 2 halo stages) or a streaming B ring;
    // after the barrier block: the EPI_MERGE db rows, then the TMA-store staging
    {
        const int stage_b = bn / cg * kBK * 4;
        const int nkb = 9 * hg.cblocks;
        hg.hstage_bytes = (hg.rows * 128 + 1023) / 1024 * 1024;
        const int db_need = p.epi.db_partial != nullptr ? 4 * ((d.N + 31) / 32 * 32) * 4 : 0;
        const bool tma = tma_store_setup(p.epi, d.M, d.N, &hg, &p.ts);
        int extra = db_need;
        const bool one_col = d.N <= bn;
        if (tma) {
            p.ts.stage_off = 1024 + (db_need + 1023) / 1024 * 1024;
            extra = p.ts.stage_off - 1024 + kEpiStageBytes;
            // masked merge: two staging boxes per warp (the next chunk's mask load
            // does not wait for the previous chunk's store) when the resident B
            // slice still fits next to 3 halo stages
            const int extra2 = p.ts.stage_off - 1024 + kEpiStageBytesDbuf;
            if (p.ts.mask && one_col && !dev_knob("PPB_NO_MASK_DBUF") &&
                nkb * stage_b + 3 * hg.hstage_bytes <= kHaloSmemMax - kHaloReserve - extra2) {
                p.ts.dbuf = 1;
                extra = extra2;
            }
        }
        const int avail = kHaloSmemMax - kHaloReserve - extra;
        if (one_col && nkb * stage_b + 2 * hg.hstage_bytes <= avail && !dev_knob("PPB_HALO_STREAM_B")) {
            hg.resident = 1;
            hg.bstages = nkb;
            hg.hstages = (avail - nkb * stage_b) / hg.hstage_bytes;
            if (hg.hstages > 4) hg.hstages = 4;
        } else {
            hg.resident = 0;
            hg.hstages = 3;
            hg.bstages = (avail - 3 * hg.hstage_bytes) / stage_b;
            if (hg.bstages > 12) hg.bstages = 12;
            if (hg.bstages < 2) {
                snprintf(err, errlen, "halo conv: shared memory too small for tile width %d", bn);
                return false;
            }
        }
        hg.smem = 1024 + hg.hstages * hg.hstage_bytes + hg.bstages * stage_b + 1024 + extra;
        if (2 * (hg.hstages + hg.bstages + 4) * 8 + 8 > 1024) {
            snprintf(err, errlen, "halo conv: too many pipeline barriers");
            return false;
        }
    }
    const int tm = kBM * cg;
    const long long tiles = ((hg.Mp + tm - 1) / tm) * ((d.N + bn - 1) / bn);
    const int units = sm_count() / cg;
    p.grid = static_cast<int>(tiles < units ? tiles : units) * cg;
    // A: the padded tensor as a 2-D [Mp rows][ch] matrix, box {32 ch, halo rows}
    if (!encode_map(&p.ta, d.a.ptr, static_cast<int>(hg.Mp), d.a.ch, d.a.ld, hg.rows, false, err, errlen))
        return false;
    if (d.b.geom.mode != OP_DENSE) {
        if (!encode_conv_map(&p.tb, d.b, err, errlen)) return false;
    } else if (!encode_map(&p.tb, d.b.ptr, d.b.rows, d.b.cols, d.b.ld, d.b.mn_major ? 32 : bn / cg, d.b.mn_major, err,
                           errlen)) {
        return false;
    }
    *out = p;
    return true;
}

cudaError_t halo_conv_launch(const TcGemmPlan& p, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0) return cudaSuccess;
    return p.b_mn ? launch_halo_bn<true>(p, s) : launch_halo_bn<false>(p, s);
}

}  // namespace ppb
