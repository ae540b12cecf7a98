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
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dev_knobs.h"
#include "dense_conv.cuh"
#include "epilogue.cuh"
#include "gemm_tc.h"
#include "ptx.cuh"
#include "tc_common.cuh"

#include "gemm_tc_kernel.cuh"

namespace ppb {

namespace {
std::atomic<unsigned> g_attr_set{0};  // one bit per device: smem attributes set
}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        }
    });
    return fn;
}

// Encode a 2-D fp32 map over a row-major (rows x cols, ld) matrix whose
// innermost (contiguous) dimension is `cols`, box {32, box_rows}.
bool encode_map(CUtensorMap* map, const float* ptr, int rows, int cols, long long ld,
                int box_rows, bool mn_major, char* err, size_t errlen) {
    auto enc = get_encode();
    if (enc == nullptr) {
        snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    if ((reinterpret_cast<uintptr_t>(ptr) & 15u) != 0 || (ld * 4) % 16 != 0) {
        snprintf(err, errlen, "TMA operand not 16-byte aligned (ptr=%p ld=%lld)", (const void*)ptr, ld);
        return false;
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
    cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        snprintf(err, errlen, "cuTensorMapEncodeTiled failed (%d) rows=%d cols=%d ld=%lld box=%d",
                 static_cast<int>(r), rows, cols, ld, box_rows);
        return false;
    }
    return true;
}

// Rank-3/4 map for implicit-GEMM conv operands (see gemm.h): a padded NHWC
// tensor {ch, wp, hp, imgs} (pitch ld) or a [u][taps][ck] weight tensor.
bool encode_conv_map(CUtensorMap* map, const Operand& o, char* err, size_t errlen) {
    auto enc = get_encode();
    if (enc == nullptr) {
        snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable");
        return false;
    }
    if ((reinterpret_cast<uintptr_t>(o.ptr) & 15u) != 0 || (o.ld * 4) % 16 != 0) {
        snprintf(err, errlen, "TMA conv operand not 16-byte aligned (ld=%lld)", o.ld);
        return false;
    }
    const ConvGeom& g = o.geom;
    cuuint64_t dims[4];
    cuuint64_t strides[3];
    cuuint32_t box[4];
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    cuuint32_t rank;
    if (g.mode == OP_WFLIP) {
        rank = 3;
        dims[0] = o.ch;
        dims[1] = o.wp;
        dims[2] = o.hp;
        strides[0] = o.ld * 4;
        strides[1] = static_cast<cuuint64_t>(o.wp) * o.ld * 4;
        box[0] = 32;
        box[1] = 1;
        box[2] = 32;
    } else {
        rank = 4;
        dims[0] = o.ch;
        dims[1] = o.wp;
        dims[2] = o.hp;
        dims[3] = o.imgs;
        strides[0] = o.ld * 4;
        strides[1] = static_cast<cuuint64_t>(o.wp) * o.ld * 4;
        strides[2] = static_cast<cuuint64_t>(o.hp) * o.wp * o.ld * 4;
        box[0] = 32;
        box[1] = g.bw;
        box[2] = g.bh + (g.rr ? g.ksz - 1 : 0);
        box[3] = g.bn;
    }
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(o.ptr), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     o.mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        snprintf(err, errlen, "cuTensorMapEncodeTiled (conv, mode %d) failed (%d)", g.mode, static_cast<int>(r));
        return false;
    }
    return true;
}

// ---------------------------------------------------------------- TMA-store epilogue setup

// EPI_MERGE through a 2x2 pool (tc kernel rows = pooled pixels): the
// error-signal map traverses the full grid with element stride 2 in w and h,
// so the box of 32 pooled pixels' quadrant q lands on positions
// (2y + dy, 2x + dx); the mask map covers the pooled activation.
static bool tma_store_setup_pool2(const EpiParams& e, int M, int N, TmaStore* ts) {
    auto enc = get_encode();
    static const bool off = dev_knob("PPB_NO_TMA_POOL2");
    if (off || enc == nullptr || N % 32 != 0 || M <= 0 || e.mg_dld % 4 != 0 || e.mg_uch % 4 != 0 ||
        (reinterpret_cast<uintptr_t>(e.mg_argmax) & 3u) != 0)
        return false;
    const int wo = e.mg_wg, ho = e.mg_hg, pix = wo * ho;
    if (pix <= 0 || M % pix != 0 || 2 * wo > 256 || 2 * ho > 256) return false;
    cuuint32_t box[4] = {32u, 32u, 1u, 1u};
    if (wo >= 32) {
        if (wo % 32 != 0) return false;
    } else if (32 % wo != 0) {
        return false;
    } else if (pix >= 32) {
        if (pix % 32 != 0) return false;
        box[1] = wo;
        box[2] = 32 / wo;
    } else {
        if (32 % pix != 0) return false;
        box[1] = wo;
        box[2] = ho;
        box[3] = 32 / pix;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, e.mg_d) != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != dev) {
        cudaGetLastError();
        return false;
    }
    if ((reinterpret_cast<uintptr_t>(e.mg_d) & 15u) != 0) return false;
    const long long ld = e.mg_dld;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(2 * wo), static_cast<cuuint64_t>(2 * ho),
                          static_cast<cuuint64_t>(M / pix)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 4, static_cast<cuuint64_t>(e.mg_dwp) * ld * 4,
                             static_cast<cuuint64_t>(e.mg_dhp) * e.mg_dwp * ld * 4};
    cuuint32_t sbox[4] = {32u, 2 * box[1], 2 * box[2], box[3]};
    cuuint32_t sestr[4] = {1u, 2u, 2u, 1u};
    float* base = e.mg_d + (static_cast<long long>(e.mg_dpad) * e.mg_dwp + e.mg_dpad) * ld;
    if (enc(&ts->map[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, sbox, sestr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    ts->mask = 0;
    if (e.mg_mask != nullptr) {
        const float* mptr = e.mg_mask + e.mg_mcol0;
        const long long mld = e.mg_mld;
        if ((reinterpret_cast<uintptr_t>(mptr) & 15u) != 0 || mld % 4 != 0) return false;
        cuuint64_t mdims[4] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(wo), static_cast<cuuint64_t>(ho),
                               static_cast<cuuint64_t>(M / pix)};
        cuuint64_t mstr[3] = {static_cast<cuuint64_t>(mld) * 4, static_cast<cuuint64_t>(e.mg_mwp) * mld * 4,
                              static_cast<cuuint64_t>(e.mg_mhp) * e.mg_mwp * mld * 4};
        cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
        const float* mbase = mptr + (static_cast<long long>(e.mg_mpad) * e.mg_mwp + e.mg_mpad) * mld;
        if (enc(&ts->mmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(mbase), mdims, mstr, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        ts->mask = 1;
    }
    ts->rank = 4;
    ts->wo = wo;
    ts->pix = pix;
    ts->segw = 0;
    ts->pool2 = 1;
    ts->n = 1;
    return true;
}

bool tma_store_setup(const EpiParams& e, int M, int N, const HaloGeom* hg, TmaStore* ts) {
    ts->mask_pf = dev_knob("PPB_NO_MASK_PREFETCH") ? 0 : 1;  // A/B switch (DEV builds)
    ts->n = 0;
    ts->pool2 = 0;
    static const bool off = dev_knob("PPB_NO_TMA_STORE");
    auto enc = get_encode();
    if (off || enc == nullptr || N < 32 || M <= 0) return false;
    if (e.mode == EPI_MERGE && e.mg_pool == 2) return hg == nullptr && tma_store_setup_pool2(e, M, N, ts);
    float* ptrs[kMaxDst];
    int nd = 0;
    long long ld = 0;
    int col0 = 0;
    bool padded = false;
    int hp = 1, wp = 1, pad = 0, wo = 1, ho = 1;
    switch (e.mode) {
        case EPI_STORE:
            for (int d = 0; d < e.ndst; ++d) ptrs[nd++] = e.dst[d];
            ld = e.ldd;
            col0 = e.col0;
            if (e.remap) {
                padded = true;
                hp = e.r_hp, wp = e.r_wp, pad = e.r_pad, wo = e.r_wo, ho = e.r_howo / e.r_wo;
            }
            break;
        case EPI_MERGE:
            if (e.mg_pool != 1 || N % 32 != 0) return false;
            if (e.mg_mask != nullptr && (e.mg_mld % 4 != 0 || e.mg_mcol0 % 4 != 0 ||
                                         (reinterpret_cast<uintptr_t>(e.mg_mask) & 15u) != 0))
                return false;
            ptrs[nd++] = e.mg_d;
            ld = e.mg_dld;
            padded = true;
            hp = e.mg_dhp, wp = e.mg_dwp, pad = e.mg_dpad, wo = e.mg_wg, ho = e.mg_hg;
            break;
        case EPI_MASK:
            if (N % 32 != 0 || e.ldm % 4 != 0 || e.mcol0 % 4 != 0 || (reinterpret_cast<uintptr_t>(e.mask) & 15u) != 0)
                return false;
            ptrs[nd++] = e.dst[0];
            ld = e.ldd;
            col0 = e.col0;
            break;
        default:
            return false;
    }
    if (nd == 0 || ld % 4 != 0 || col0 % 4 != 0) return false;
    // Shards of one layer store disjoint column ranges of the same rows
    // concurrently; a bulk tensor store that shares a 32 B sector with another
    // writer's range corrupts it (measured: LeNet 120 -> 60/60 shards), so the
    // TMA path needs sector-aligned ranges unless this GEMM owns whole rows.
    const bool whole_rows = col0 == 0 && (N + 3) / 4 * 4 == ld;
    if (!whole_rows && e.seg_w == 0 && (col0 % 8 != 0 || N % 8 != 0 || ld % 8 != 0)) return false;
    int dev = 0;
    cudaGetDevice(&dev);
    for (int d = 0; d < nd; ++d) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptrs[d]) != cudaSuccess || a.type != cudaMemoryTypeDevice || a.device != dev) {
            cudaGetLastError();
            return false;  // peer destinations keep the register path
        }
        if ((reinterpret_cast<uintptr_t>(ptrs[d] + col0) & 15u) != 0) return false;
    }
    cuuint64_t dims[4];
    cuuint64_t strides[3];
    cuuint32_t box[4] = {32u, 32u, 1u, 1u};
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    cuuint32_t rank = 2;
    long long base_off = col0;
    ts->segw = 0;
    if (e.mode == EPI_STORE && e.seg_w > 0) {  // dense conv: {c, p, row}, box {32, 1, 32}
        if (hg != nullptr || padded || e.seg_w % 32 != 0 || N % e.seg_w != 0 || e.seg_pitch % 8 != 0 || col0 % 8 != 0 ||
            ld % 8 != 0)
            return false;
        rank = 3;
        dims[0] = static_cast<cuuint64_t>(e.seg_w);
        dims[1] = static_cast<cuuint64_t>(N / e.seg_w);
        dims[2] = static_cast<cuuint64_t>(M);
        strides[0] = static_cast<cuuint64_t>(e.seg_pitch) * 4;
        strides[1] = static_cast<cuuint64_t>(ld) * 4;
        box[1] = 1;
        box[2] = 32;
        ts->segw = e.seg_w;
    } else if (hg != nullptr) {
        // halo rows are padded positions: identity when the destination has the same grid
        if (!padded || hp != hg->hp || wp != hg->wp || pad != 1 || ho != hg->ho || wo != hg->wo) return false;
        dims[0] = static_cast<cuuint64_t>(N);
        dims[1] = static_cast<cuuint64_t>(hg->Mp);
        strides[0] = static_cast<cuuint64_t>(ld) * 4;
    } else if (!padded) {
        dims[0] = static_cast<cuuint64_t>(N);
        dims[1] = static_cast<cuuint64_t>(M);
        strides[0] = static_cast<cuuint64_t>(ld) * 4;
    } else {
        const int pix = wo * ho;
        if (pix <= 0 || M % pix != 0) return false;
        rank = 4;
        if (wo >= 32) {
            if (wo % 32 != 0) return false;
            box[1] = 32;
        } else if (32 % wo != 0) {
            return false;
        } else if (pix >= 32) {
            if (pix % 32 != 0) return false;
            box[1] = wo;
            box[2] = 32 / wo;
        } else {
            if (32 % pix != 0) return false;
            box[1] = wo;
            box[2] = ho;
            box[3] = 32 / pix;
        }
        dims[0] = static_cast<cuuint64_t>(N);
        dims[1] = static_cast<cuuint64_t>(wo);
        dims[2] = static_cast<cuuint64_t>(ho);
        dims[3] = static_cast<cuuint64_t>(M / pix);
        strides[0] = static_cast<cuuint64_t>(ld) * 4;
        strides[1] = static_cast<cuuint64_t>(wp) * ld * 4;
        strides[2] = static_cast<cuuint64_t>(hp) * wp * ld * 4;
        base_off += (static_cast<long long>(pad) * wp + pad) * ld;
        ts->wo = wo;
        ts->pix = pix;
    }
    // mask map (EPI_MERGE pool 1 / EPI_MASK): the activation at the same rows / columns
    const float* mptr = nullptr;
    long long mld = 0;
    if (e.mode == EPI_MERGE && e.mg_mask != nullptr) {
        mptr = e.mg_mask + e.mg_mcol0;
        mld = e.mg_mld;
        if (hg != nullptr ? (e.mg_mhp != hg->hp || e.mg_mwp != hg->wp || e.mg_mpad != 1)
                          : (e.mg_mhp != hp || e.mg_mwp != wp || e.mg_mpad != pad))
            return false;
    } else if (e.mode == EPI_MASK) {
        mptr = e.mask + e.mcol0;
        mld = e.ldm;
    }
    // residual layer, identity shortcut: the shortcut rows share the store's
    // padded geometry, so they load as the "mask" box (TmaStore::res)
    bool res = false;
    static const bool no_res_box = dev_knob("PPB_NO_RES_BOX");  // A/B switch
    if (e.mode == EPI_STORE && e.rs_src != nullptr && e.rs_f == 1 && e.remap && !no_res_box &&
        e.rs_C - e.rs_col0 >= N && (hg != nullptr ? (e.rs_hp == hg->hp && e.rs_wp == hg->wp && e.rs_pad == 1)
                                                  : (rank == 4 && e.rs_hp == hp && e.rs_wp == wp && e.rs_pad == pad))) {
        mptr = e.rs_src + e.rs_col0;
        mld = e.rs_ld;
        res = true;
    }
    ts->mask = 0;
    ts->res = 0;
    static const bool no_mask = dev_knob("PPB_NO_TMA_MASK");
    if (mptr != nullptr && no_mask) return false;
    if (mptr != nullptr) {
        if ((reinterpret_cast<uintptr_t>(mptr) & 15u) != 0 || mld % 4 != 0) return false;
        cuuint64_t mstr[3] = {static_cast<cuuint64_t>(mld) * 4, static_cast<cuuint64_t>(wp) * mld * 4,
                              static_cast<cuuint64_t>(hp) * wp * mld * 4};
        const long long moff = rank == 4 ? (static_cast<long long>(pad) * wp + pad) * mld : 0;
        if (enc(&ts->mmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(mptr) + moff, dims, mstr, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        ts->mask = 1;
        ts->res = res ? 1 : 0;
        // halo merge with a shortcut gradient of the same padded geometry: its
        // rows load as a second box (used when the kernel has two boxes per warp)
        ts->sg = 0;
        static const bool no_sg_box = dev_knob("PPB_NO_SG_BOX");  // A/B switch
        if (e.mode == EPI_MERGE && e.mg_sg != nullptr && hg != nullptr && rank == 2 && !no_sg_box &&
            e.mg_shp == hg->hp && e.mg_swp == hg->wp && e.mg_spad == 1 && e.mg_sld % 4 == 0 &&
            (reinterpret_cast<uintptr_t>(e.mg_sg + e.mg_sc0) & 15u) == 0) {
            cuuint64_t sstr[3] = {static_cast<cuuint64_t>(e.mg_sld) * 4, 0, 0};
            if (enc(&ts->smap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(e.mg_sg + e.mg_sc0), dims,
                    sstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
                ts->sg = 1;
        }
    }
    ts->rank = static_cast<int>(rank);
    for (int d = 0; d < nd; ++d) {
        CUresult r = enc(&ts->map[d], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, ptrs[d] + base_off, dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return false;
    }
    ts->n = nd;
    return true;
}

bool tma_store_setup_splitk(const SplitK& sk, int M, int N, TmaStore* ts) {
    ts->n = 0;
    static const bool off = dev_knob("PPB_NO_TMA_STORE");
    auto enc = get_encode();
    static const bool off_sk = dev_knob("PPB_NO_TMA_SPLITK");
    if (off || off_sk || enc == nullptr || (sk.splits < 2 && !sk.partial) || sk.ws == nullptr) return false;
    const int inner = sk.trans ? M : N, outer = sk.trans ? N : M;
    if (inner < 32 || sk.ld % 4 != 0 || sk.stride % 4 != 0 || (reinterpret_cast<uintptr_t>(sk.ws) & 15u) != 0)
        return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer),
                          static_cast<cuuint64_t>(sk.splits)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(sk.ld) * 4, static_cast<cuuint64_t>(sk.stride) * 4};
    cuuint32_t box[3] = {32u, 32u, 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    if (enc(&ts->map[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, sk.ws, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    ts->rank = 3;
    ts->tr = sk.trans;
    ts->n = 1;
    return true;
}

// Programmatic dependent launch is opt-in (PPB_PDL=1): with the wgrad stream
// overlapping the forward / dgrad chain, successors that launch early park
// CTAs on SMs the other stream could use (measured 2.305 ms without, 2.312 ms
// with the late trigger, 2.340 ms with an early trigger).
bool pdl_enabled() {
    return dev_knob("PPB_PDL");
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Set the dynamic shared-memory limit of every instantiation on the current
// device (must happen before any launch is captured into a CUDA graph).
cudaError_t tc_gemm_init_device() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t (*f)() : {tc_init_mn<false, false>, tc_init_mn<false, true>, tc_init_mn<true, false>,
                               tc_init_mn<true, true>})
        if (e == cudaSuccess) e = f();
    if (e == cudaSuccess) e = halo_conv_init_device();
    int dev = 0;
    cudaGetDevice(&dev);
    if (e == cudaSuccess) g_attr_set.fetch_or(1u << (dev & 31));
    return e;
}

bool tc_gemm_prepare(const GemmDesc& d, TcGemmPlan* out, int force_bn, char* err, size_t errlen,
                     const WsAlloc& ws_alloc) {
    // 3x3 convs over large padded grids: the halo-reuse kernel (conv_halo.cu)
    static const bool no_halo = dev_knob("PPB_NO_HALO");
    if (!d.partial_out && (force_bn >= 1000 || (force_bn == 0 && !no_halo && halo_conv_preferred(d))) &&
        halo_conv_eligible(d))
        return halo_conv_prepare(d, out, force_bn, err, errlen);
    if (force_bn >= 1000) {
        snprintf(err, errlen, "halo conv tile forced on an ineligible GEMM");
        return false;
    }
    if (force_bn == 0 && ws_alloc && wgrad_halo_eligible(d)) return wgrad_halo_prepare(d, out, err, errlen, ws_alloc);
    TcGemmPlan p;
    p.M = d.M;
    p.N = d.N;
    p.K = d.K;
    p.a_mn = d.a.mn_major;
    p.b_mn = d.b.mn_major;
    p.epi = d.epi;
    p.epi.M = d.M;
    p.epi.N = d.N;
    p.epi.dbg = static_cast<int>(dev_knob_uint("PPB_GEMM_DBG"));  // timing probes only
    if (d.K < 1) {
        snprintf(err, errlen, "GEMM with K=%d", d.K);
        return false;
    }
    const int sms = sm_count();
    const int nk = (d.K + kBK - 1) / kBK;
    const bool can_split = static_cast<bool>(ws_alloc) && nk >= 16;
    // Split count that fills the SMs for a tile grid (>= 8 K blocks per split).
    auto splits_for = [&](int tiles, int units) {
        if (!can_split || tiles >= units) return 1;
        int sp = units / tiles;
        if (sp > nk / 8) sp = nk / 8;
        if (sp > sms) sp = sms;
        return sp < 1 ? 1 : sp;
    };
    // force_bn: 0 = auto; 64/128/256 = 1-CTA tiles of that width;
    // -128/-256 = CTA-pair tiles (256 x |bn|).
    int bn = 256, cg = 1;
    int best_sp = -1;  // split count chosen with the tile shape (-1: splits_for)
    if (force_bn == 64 || force_bn == 128 || force_bn == 256) {
        bn = force_bn;
    } else if (force_bn == -64 || force_bn == -128 || force_bn == -256) {
        bn = -force_bn;
        cg = 2;
    } else {
        // Score each tile shape by (relative MMA efficiency of the shape,
        // measured on the wide-MLP GEMM) x (fraction of the tile that is
        // real output) x (wave fill after split-K); keep the best.
        struct Cand {
            int cg, bn;
            double eff;
        };
        // (an operand-bound table {1, .69, .69, .52, .35} measured slower on the
        // VGG step, 2.30 vs 2.27 ms: the split-K reduction it then prefers
        // costs more than the model charges)
        // CTA-pair 64-wide tiles: each SM reads its 128 A rows and HALF of B
        // from shared memory (the pair exchanges B), 5 instead of 6 KB per
        // 128 x 64 x 8 MMA, so the narrow layers' operand-rate cap
        // rises by ~1.2x
        const Cand cands_std[] = {{2, 256, 1.0}, {2, 128, 0.85}, {1, 256, 0.93}, {1, 128, 0.8}, {2, 64, 0.62},
                                  {1, 64, 0.55}};
        const Cand cands_op[] = {{2, 256, 1.0}, {2, 128, 0.69}, {1, 256, 0.69}, {1, 128, 0.52}, {2, 64, 0.42},
                                 {1, 64, 0.35}};
        // wgrad + SGD (reduction free as a side job): the operand-bound table
        // picks slightly better tiles (2.238 -> 2.233 ms); elsewhere it prefers
        // split-K whose reduction costs more than modelled
        static const bool sgd_std = dev_knob("PPB_SGD_STDTABLE");
        const Cand* cands = (!sgd_std && d.epi.mode == EPI_SGD) ? cands_op : cands_std;
        double best = -1;
        static const bool no_pair64 = dev_knob("PPB_NO_PAIR64");  // A/B switch
        for (int ci = 0; ci < 6; ++ci) {
            const Cand& c = cands[ci];
            if (no_pair64 && c.cg == 2 && c.bn == 64) continue;
            if (c.cg == 2 && d.M <= 128) continue;
            const int tm = kBM * c.cg;
            const int num_m = (d.M + tm - 1) / tm, num_n = (d.N + c.bn - 1) / c.bn;
            const int tiles = num_m * num_n, units = sms / c.cg;
            const double frac = static_cast<double>(d.M) / (num_m * tm) * static_cast<double>(d.N) / (num_n * c.bn);
            // with and without split-K
            for (int sp : {1, splits_for(tiles, units)}) {
                const int work = tiles * sp;
                const int waves = (work + units - 1) / units;
                const double fill = static_cast<double>(work) / (static_cast<double>(waves) * units);
                // estimated time: MMA at the shape's efficiency, plus the split-K
                // reduction pass (partials re-read from L2 + the epilogue's write +
                // a launch) unless it is a wgrad+SGD, whose reduction rides in the
                // next GEMM's mainloop (SideJob)
                double t = 2.0 * d.M * d.N * d.K / (806e12 * c.eff * fill * frac);
                if (sp > 1 && d.epi.mode != EPI_SGD) t += (sp + 1.0) * d.M * d.N * 4.0 / 8e12 + 3e-6;
                const double score = 1.0 / t;
                if (score > best * (1.0 + 1e-9)) {
                    best = score;
                    cg = c.cg;
                    bn = c.bn;
                    best_sp = sp;
                }
            }
        }
    }
    // A/B probe (DEV builds): PPB_FORCE_TILE="M,N,K,cg,bn,splits[;...]" forces
    // the tiling of every GEMM of that shape (splits 0 = keep the chooser's)
    if (const char* ft = dev_knob("PPB_FORCE_TILE") ? getenv("PPB_FORCE_TILE") : nullptr) {
        int fm, fn, fk, fcg, fbn, fsp, used = 0;
        for (const char* q = ft; sscanf(q, "%d,%d,%d,%d,%d,%d%n", &fm, &fn, &fk, &fcg, &fbn, &fsp, &used) == 6;) {
            if (fm == d.M && fn == d.N && fk == d.K) {
                cg = fcg;
                bn = fbn;
                best_sp = fsp > 0 ? fsp : -1;
            }
            q += used;
            if (*q != ';') break;
            ++q;
        }
    }
    // A/B probe (DEV builds): CTA-pair tiles for narrow wgrads (fewer M tiles,
    // so the error signal is re-read fewer times through L2)
    if (force_bn == 0 && cg == 1 && bn == 64 && d.epi.mode == EPI_SGD && d.M > 128 && dev_knob("PPB_WGRAD_PAIR")) {
        cg = 2;
        best_sp = -1;
    }
    p.bn = bn;
    p.cg = cg;
    const int tiles = ((d.M + kBM * cg - 1) / (kBM * cg)) * ((d.N + bn - 1) / bn);
    const int units = sms / cg;
    // Split-K when the output tiles cannot fill the SMs (e.g. conv wgrad:
    // small C_out x 9*C_in output, K = every pixel of the batch); partial
    // sums are reduced in split order (deterministic).
    {
        int splits = d.force_splits > 0 ? d.force_splits : best_sp > 0 ? best_sp : splits_for(tiles, units);
        if (splits > nk) splits = nk;
        if (d.partial_out && !ws_alloc) {
            snprintf(err, errlen, "partial-sum GEMM without a workspace");
            return false;
        }
        if (splits >= 2 || d.partial_out) {
            const int kps = (nk + splits - 1) / splits;
            splits = (nk + kps - 1) / kps;
            p.sk.splits = splits;
            p.sk.kps = kps;
            p.sk.trans = d.epi.mode == EPI_SGD && d.epi.sgd_t ? 1 : 0;
            p.sk.ld = p.sk.trans ? (d.M + 3) / 4 * 4 : (d.N + 3) / 4 * 4;
            p.sk.stride = p.sk.ld * (p.sk.trans ? d.N : d.M);
            p.sk.ws = ws_alloc(static_cast<size_t>(p.sk.stride) * splits);
            if (p.sk.ws == nullptr) {
                snprintf(err, errlen, "split-K workspace allocation failed");
                return false;
            }
            // in-kernel fixup: measured slower than the reduction kernel (the
            // last warp's serial row-per-thread reads sit on the tile's tail:
            // VGG step 2.54 -> 3.07 ms), so opt-in only
            const bool fixup_on = dev_knob("PPB_SPLITK_FIXUP");
            p.sk.partial = d.partial_out;
            if (splits <= 8 && fixup_on && !d.partial_out) {
                const size_t nctr = static_cast<size_t>(tiles) * cg * 8;
                float* c = ws_alloc(nctr);
                if (c != nullptr && cudaMemset(c, 0, nctr * sizeof(int)) == cudaSuccess) {
                    p.sk.counters = reinterpret_cast<int*>(c);
                    p.sk.fixup = 1;
                }
            }
        }
    }
    const int work = tiles * p.sk.splits;
    p.grid = (work < units ? work : units) * cg;
    // shared memory: stage ring + barrier block, then the EPI_MERGE db rows,
    // then the TMA-store staging; the ring gives up stages (down to 4) to fit
    // row reuse for 3x3 implicit convs whose 128-row tiles are whole image
    // rows of one image: one A box of bh + 2 rows per (column tap, channel
    // block) feeds the 3 row taps, so A crosses L2 -> SM 3x instead of 9x
    // (conv2 forward: 1.5 GB of L2 reads for 0.17 GB of activations)
    const ConvGeom& ag = d.a.geom;
    static const bool no_rr = dev_knob("PPB_NO_ROW_REUSE");  // A/B switch
    const bool rr = !no_rr && ag.mode == OP_CONV_ROWS && !d.a.mn_major && ag.ksz == 3 && ag.bn == 1 &&
                    ag.bw % 8 == 0 && ag.bh + ag.ksz - 1 <= 256 && p.sk.splits == 1 && !p.sk.partial &&
                    !d.partial_out;
    const int stage_b = bn / cg * kBK * 4;
    const int stage_bytes = rr ? (ag.bh + ag.ksz - 1) * ag.bw * 128 + ag.ksz * stage_b : kBM * kBK * 4 + stage_b;
    const int def_stages = (200 * 1024) / stage_bytes > 8 ? 8 : (200 * 1024) / stage_bytes;
    p.stage_bytes = stage_bytes;
    constexpr int kCapSmem = 227 * 1024;
    auto ring = [&](int st) { return 1024 + st * stage_bytes + 256; };
    p.stages = def_stages;
    if (p.epi.db_partial != nullptr) {  // in-epilogue bias partials: single-pass (no split-K) only
        const int need = 8 * ((d.N + 31) / 32 * 32) * 4;  // one row per epilogue warp
        if (p.sk.splits > 1 || ring(p.stages) + need > kCapSmem) p.epi.db_partial = nullptr;
        else p.db_smem = need;
    }
    if (p.sk.splits == 1 && !p.sk.partial ? tma_store_setup(p.epi, d.M, d.N, nullptr, &p.ts)
                         : tma_store_setup_splitk(p.sk, d.M, d.N, &p.ts)) {
        // staging after the barrier block and the db rows, 1 KB aligned (SW128 boxes)
        const int off = 1024 + (p.db_smem + 1023) / 1024 * 1024;
        const int extra = off + kEpiStageBytes - 256;
        int st = p.stages;
        while (ring(st) + extra > kCapSmem && st > 4) --st;
        static const bool no_dbuf = dev_knob("PPB_NO_STAGE_DBUF");  // A/B switch
        if (ring(st) + extra <= kCapSmem) {
            p.stages = st;
            p.ts.stage_off = off;
            p.db_smem = extra;
            // second staging set when it fits without giving up ring stages
            // (plain stores / split-K partials: the masked, pooled-merge and
            // pool-from-staging epilogues read their box back)
            const int extra2 = off + kEpiStageBytesDbuf - 256;
            // a short K loop (conv1: one K block per tile) needs few ring
            // stages; there the second staging set is worth more (each chunk
            // otherwise waits for the previous chunk's bulk store to read its box)
            const int kpt = p.sk.splits > 1 || p.sk.partial ? p.sk.kps : nk;
            int st2 = st;
            while (ring(st2) + extra2 > kCapSmem && st2 > 4 && st2 > 2 * kpt) --st2;
            if (!p.ts.mask && !p.ts.pool2 && p.epi.pl_on != 2 && p.epi.pl_on != 3 && ring(st2) + extra2 <= kCapSmem &&
                !no_dbuf) {
                p.stages = st2;
                p.ts.dbuf = 1;
                p.db_smem = extra2;
            }
        } else {
            p.ts = TmaStore{};
        }
    }
    // A: M extent x K.  K-major: rows=M, cols=K, box {32, 128}.  MN-major:
    // stored K x M (rows=K, cols=M), box {32, 32}.  B rows per CTA = bn / cg.
    p.ga = d.a.geom;
    p.ga.rr = rr ? 1 : 0;
    p.gb = d.b.geom;
    if (d.a.geom.mode != OP_DENSE) {
        Operand a = d.a;
        a.geom.rr = p.ga.rr;
        if (!encode_conv_map(&p.ta, a, err, errlen)) return false;
    } else if (!encode_map(&p.ta, d.a.ptr, d.a.rows, d.a.cols, d.a.ld, d.a.mn_major ? 32 : kBM, d.a.mn_major, err,
                           errlen)) {
        return false;
    }
    if (d.b.geom.mode != OP_DENSE) {
        if (d.b.geom.mode == OP_CONV_ROWS) {
            snprintf(err, errlen, "conv pixel rows are only supported as operand A");
            return false;
        }
        if (!encode_conv_map(&p.tb, d.b, err, errlen)) return false;
    } else if (!encode_map(&p.tb, d.b.ptr, d.b.rows, d.b.cols, d.b.ld, d.b.mn_major ? 32 : bn / cg, d.b.mn_major,
                           err, errlen)) {
        return false;
    }
    *out = p;
    return true;
}

cudaError_t tc_gemm_launch_reduce(const TcGemmPlan& p, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0) return cudaSuccess;
    return launch_splitk_reduce(p, s);
}

cudaError_t tc_gemm_launch(const TcGemmPlan& p, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0) return cudaSuccess;
    if (p.halo == 2) return wgrad_halo_launch(p, s);
    if (p.halo) return halo_conv_launch(p, s);
    int dev = 0;
    cudaGetDevice(&dev);
    if ((g_attr_set.load() & (1u << (dev & 31))) == 0) {
        cudaError_t e = tc_gemm_init_device();
        if (e != cudaSuccess) return e;
    }
    if (p.a_mn) return p.b_mn ? tc_launch_mn<true, true>(p, s) : tc_launch_mn<true, false>(p, s);
    return p.b_mn ? tc_launch_mn<false, true>(p, s) : tc_launch_mn<false, false>(p, s);
}

}  // namespace ppb