// Exact-fp32 shard GEMM on the CUDA cores: every output is one fp32 FMA chain
// over k in ascending order (the reference's summation order, tinynet.cpp:11-48,
// carried out in fp32).  Same operand conventions and fused epilogues as the
// tcgen05 kernel; used for the tight-tolerance parity mode and as a
// cross-check of the tensor-core path, never on the benchmarked path.
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "gemm_tc.h"

namespace ppb {

namespace {

constexpr int kRows = 64;  // rows per block, one per thread
constexpr int kCols = 32;  // columns per block (one epilogue chunk)
constexpr int kK = 32;

__global__ void __launch_bounds__(kRows) simt_gemm_kernel(const float* __restrict__ a, long long lda,
                                                           bool a_mn, const float* __restrict__ b,
                                                           long long ldb, bool b_mn, int M, int N,
                                                           int K, const __grid_constant__ EpiParams epi) {
    __shared__ float sa[kRows][kK + 1];
    __shared__ float sb[kCols][kK + 1];
    const int t = threadIdx.x;
    const int m0 = blockIdx.x * kRows;
    const int n0 = blockIdx.y * kCols;
    float acc[kCols];
#pragma unroll
    for (int i = 0; i < kCols; ++i) acc[i] = 0.f;

    for (int k0 = 0; k0 < K; k0 += kK) {
        // A tile: kRows x kK
        for (int idx = t; idx < kRows * kK; idx += kRows) {
            const int r = idx / kK, c = idx % kK;
            const int m = m0 + r, k = k0 + c;
            float v = 0.f;
            if (m < M && k < K) v = a_mn ? a[static_cast<long long>(k) * lda + m] : a[static_cast<long long>(m) * lda + k];
            sa[r][c] = v;
        }
        for (int idx = t; idx < kCols * kK; idx += kRows) {
            const int r = idx / kK, c = idx % kK;
            const int n = n0 + r, k = k0 + c;
            float v = 0.f;
            if (n < N && k < K) v = b_mn ? b[static_cast<long long>(k) * ldb + n] : b[static_cast<long long>(n) * ldb + k];
            sb[r][c] = v;
        }
        __syncthreads();
        const int kend = K - k0 < kK ? K - k0 : kK;
        for (int k = 0; k < kend; ++k) {
            const float av = sa[t][k];
#pragma unroll
            for (int i = 0; i < kCols; ++i) acc[i] = fmaf(av, sb[i][k], acc[i]);
        }
        __syncthreads();
    }
    epilogue32(epi, m0 + t, n0, acc);
}

}  // namespace

cudaError_t simt_gemm_launch(const GemmDesc& d, cudaStream_t s) {
    if (d.M <= 0 || d.N <= 0) return cudaSuccess;
    EpiParams epi = d.epi;
    epi.M = d.M;
    epi.N = d.N;
    dim3 grid((d.M + kRows - 1) / kRows, (d.N + kCols - 1) / kCols);
    simt_gemm_kernel<<<grid, kRows, 0, s>>>(d.a.ptr, d.a.ld, d.a.mn_major, d.b.ptr, d.b.ld,
                                            d.b.mn_major, d.M, d.N, d.K, epi);
    return cudaGetLastError();
}

}  // namespace ppb
