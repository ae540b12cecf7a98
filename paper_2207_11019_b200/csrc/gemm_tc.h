#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>

#include "gemm.h"
#include "tma_epi.cuh"

namespace ppb {

// A shard GEMM with its TMA descriptors encoded once (at session build), so a
// step is launch-only.
struct TcGemmPlan {
    CUtensorMap ta;
    CUtensorMap tb;
    int M = 0, N = 0, K = 0;
    int bn = 256;
    int cg = 1;  // 1: single-CTA 128-row tiles, 2: CTA-pair 256-row tiles
    int grid = 1;
    bool a_mn = false, b_mn = false;
    EpiParams epi;
    ConvGeom ga, gb;
    SplitK sk;
    int halo = 0;  // 1: conv_halo.cu kernel (hg describes the padded grid); 2: wgrad_halo.cu kernel (wg)
    int db_smem = 0;  // extra dynamic smem past the ring: EPI_MERGE db rows + TMA-store staging
    int stages = 0;   // tc_gemm ring stages (<= TcCfg::kStages)
    int stage_bytes = 0;  // tc_gemm bytes per ring stage (A + B; larger with row reuse)
    HaloGeom hg;
    WgradGeom wg;
    TmaStore ts;  // TMA-store epilogue (ts.n == 0: register epilogue)
    SideJob sj;   // a previous GEMM's deferred split-K reduction
};

// ws_alloc (optional): allocates split-K workspace (floats) on the GEMM's
// device; without it the GEMM never splits K.
using WsAlloc = std::function<float*(size_t)>;
bool tc_gemm_prepare(const GemmDesc& d, TcGemmPlan* out, int force_bn, char* err, size_t errlen,
                     const WsAlloc& ws_alloc = nullptr);
cudaError_t tc_gemm_launch(const TcGemmPlan& p, cudaStream_t s);
// The reduction + epilogue of a partial-sum plan on its own: p.sk.splits
// slices at p.sk.ws summed in slice order, then p.epi (and the bias job).
cudaError_t tc_gemm_launch_reduce(const TcGemmPlan& p, cudaStream_t s);
cudaError_t tc_gemm_init_device();
// 3x3 / 64 -> 64-channel conv weight gradients (wgrad_halo.cu)
bool wgrad_halo_eligible(const GemmDesc& d);
bool wgrad_halo_prepare(const GemmDesc& d, TcGemmPlan* out, char* err, size_t errlen, const WsAlloc& ws_alloc);
cudaError_t wgrad_halo_launch(const TcGemmPlan& p, cudaStream_t s);
// per operand-major combination (gemm_tc_inst_*.cu): launch / smem attributes
template <bool A_MN, bool B_MN>
cudaError_t tc_launch_mn(const TcGemmPlan& p, cudaStream_t s);
template <bool A_MN, bool B_MN>
cudaError_t tc_init_mn();
#define PPB_TC_DECL(A, B)                                                     \
    template <>                                                               \
    cudaError_t tc_launch_mn<A, B>(const TcGemmPlan& p, cudaStream_t s);      \
    template <>                                                               \
    cudaError_t tc_init_mn<A, B>();
PPB_TC_DECL(false, false)
PPB_TC_DECL(false, true)
PPB_TC_DECL(true, false)
PPB_TC_DECL(true, true)
#undef PPB_TC_DECL

// Halo-reuse implicit conv (conv_halo.cu): a 3x3 stride-1 conv over a padded
// NHWC grid computed in padded-position space; see halo_conv_prepare.
bool halo_conv_eligible(const GemmDesc& d);
bool halo_conv_preferred(const GemmDesc& d);  // automatic choice among eligible descriptors
bool halo_conv_prepare(const GemmDesc& d, TcGemmPlan* p, int force, char* err, size_t errlen);
cudaError_t halo_conv_launch(const TcGemmPlan& p, cudaStream_t s);
cudaError_t halo_conv_init_device();

// host helpers shared by the tcgen05 kernels (gemm_tc.cu)
bool encode_map(CUtensorMap* map, const float* ptr, int rows, int cols, long long ld, int box_rows, bool mn_major,
                char* err, size_t errlen);
bool encode_conv_map(CUtensorMap* map, const Operand& o, char* err, size_t errlen);
int sm_count();

// Exact-fp32 SIMT path with identical operand conventions and epilogues
// (debug / tight-tolerance parity mode).
cudaError_t simt_gemm_launch(const GemmDesc& d, cudaStream_t s);


}  // namespace ppb
