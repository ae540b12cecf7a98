#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>

#include "gemm.h"

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
};

// ws_alloc (optional): allocates split-K workspace (floats) on the GEMM's
// device; without it the GEMM never splits K.
using WsAlloc = std::function<float*(size_t)>;
bool tc_gemm_prepare(const GemmDesc& d, TcGemmPlan* out, int force_bn, char* err, size_t errlen,
                     const WsAlloc& ws_alloc = nullptr);
cudaError_t tc_gemm_launch(const TcGemmPlan& p, cudaStream_t s);
cudaError_t tc_gemm_init_device();

// Exact-fp32 SIMT path with identical operand conventions and epilogues
// (debug / tight-tolerance parity mode).
cudaError_t simt_gemm_launch(const GemmDesc& d, cudaStream_t s);

}  // namespace ppb
