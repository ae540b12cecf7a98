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

// Skinny GEMMs on the CUDA cores (exact fp32), for shards a tensor-core tile
// would mostly waste (the classifier head: 512 x 10 x 512 forward, 512 x 512 x
// 10 input gradient):
//  * N <= 32, K-major A and B: warp = output row, lanes stride K (ascending
//    k = lane, lane + 32, ...), fixed xor-butterfly across lanes; lane n then
//    applies the epilogue to C(m, n).
//  * K <= 32: thread = output element, ascending k.
// Every output goes through epilogue1, so all store / scatter / SGD modes work.
__global__ void __launch_bounds__(256) skinny_n_kernel(const float* __restrict__ a, long long lda,
                                                       const float* __restrict__ b, long long ldb, int M, int N,
                                                       int K, const __grid_constant__ EpiParams epi) {
    const int lane = threadIdx.x & 31;
    const int m = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (m >= M) return;
    float acc[32];
#pragma unroll
    for (int n = 0; n < 32; ++n) acc[n] = 0.f;
    const float* ar = a + static_cast<long long>(m) * lda;
    for (int k = lane; k < K; k += 32) {
        const float av = __ldg(ar + k);
#pragma unroll
        for (int n = 0; n < 32; ++n)
            if (n < N) acc[n] = fmaf(av, __ldg(b + static_cast<long long>(n) * ldb + k), acc[n]);
    }
#pragma unroll
    for (int n = 0; n < 32; ++n) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
    }
    float mine = 0.f;
#pragma unroll
    for (int n = 0; n < 32; ++n)
        if (n == lane) mine = acc[n];
    if (lane < N) {
        const long long row_off = epi.mode == EPI_STORE ? epi_store_row(epi, m) : 0;
        epilogue1(epi, m, lane, mine, row_off);
    }
}

__global__ void __launch_bounds__(256) small_k_kernel(const float* __restrict__ a, long long lda,
                                                      const float* __restrict__ b, long long ldb, bool b_mn, int M,
                                                      int N, int K, const __grid_constant__ EpiParams epi) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(M) * N) return;
    const int m = static_cast<int>(i / N), n = static_cast<int>(i % N);
    float acc = 0.f;
    const float* ar = a + static_cast<long long>(m) * lda;
    for (int k = 0; k < K; ++k) {
        const float bv = b_mn ? __ldg(b + static_cast<long long>(k) * ldb + n) : __ldg(b + static_cast<long long>(n) * ldb + k);
        acc = fmaf(__ldg(ar + k), bv, acc);
    }
    const long long row_off = epi.mode == EPI_STORE ? epi_store_row(epi, m) : 0;
    epilogue1(epi, m, n, acc, row_off);
}

}  // namespace

bool skinny_gemm_eligible(const GemmDesc& d) {
    if (d.a.geom.mode != OP_DENSE || d.b.geom.mode != OP_DENSE || d.a.mn_major) return false;
    if (d.epi.db_partial != nullptr || d.epi.seg_w != 0 || d.epi.pl_on || d.epi.mode == EPI_MERGE) return false;
    if (d.epi.mode == EPI_SGD) return false;  // wgrad stays on the tensor cores
    if (d.N <= 32 && !d.b.mn_major && static_cast<long long>(d.M) * 32 <= (1LL << 24)) return true;
    if (d.K <= 32 && static_cast<long long>(d.M) * d.N <= (1LL << 22)) return true;
    return false;
}

cudaError_t skinny_gemm_launch(const GemmDesc& d, cudaStream_t s) {
    if (d.M <= 0 || d.N <= 0) return cudaSuccess;
    EpiParams epi = d.epi;
    epi.M = d.M;
    epi.N = d.N;
    if (d.N <= 32 && !d.b.mn_major) {
        skinny_n_kernel<<<(d.M + 7) / 8, 256, 0, s>>>(d.a.ptr, d.a.ld, d.b.ptr, d.b.ld, d.M, d.N, d.K, epi);
    } else {
        const long long n = static_cast<long long>(d.M) * d.N;
        small_k_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(d.a.ptr, d.a.ld, d.b.ptr, d.b.ld,
                                                                              d.b.mn_major, d.M, d.N, d.K, epi);
    }
    return cudaGetLastError();
}

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
