// Probe (not part of the product library): kind::tf32 tcgen05.mma issue rate
// with A from shared memory (SS) vs A from tensor memory (TS), and TS with
// the A block copied smem -> TMEM by tcgen05.cp before every use -- does the
// narrow-N operand-rate cap of the SS form lift when A comes from
// TMEM?  One CTA per SM, one issuing thread, operands resident in smem (no
// TMA), `iters` passes over `kb` K-blocks of 32.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_2207_11019_b200/csrc tools/mma_probe.cu -o tools/_mma_probe.so
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

using namespace ppb;

namespace {

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t s_desc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(s_desc) : "memory");
}

// mode 0: SS; 1: TS (A already in TMEM); 2: TS with tcgen05.cp of A per K-block;
// mode 3 / 4: SS round-robin over 2 / 4 independent accumulators (is the
// narrow-N rate an issue cap, or the latency between dependent MMAs?)
template <int N>
__global__ void __launch_bounds__(128, 1) probe_kernel(int mode, int kb, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done_bar;
    const int warp = threadIdx.x / 32;
    // A blocks: kb x 16 KB (128 rows x 128 B), B blocks: kb x N x 128 B
    uint8_t* A = smem;
    uint8_t* B = smem + kb * 16384;
    for (int i = threadIdx.x; i < kb * (16384 + N * 128) / 4; i += blockDim.x)
        reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
    if (warp == 0) tmem_alloc(&tmem_slot, 512);
    if (threadIdx.x == 0) {
        mbar_init(&done_bar, 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t d_tmem = tmem;              // columns [0, N)
    const uint32_t a_tmem0 = tmem + 256;       // A slots: 2 x 32 columns at 256
    const uint32_t idesc = idesc_tf32(N, false, false);
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < kb; ++k) {
                const uint32_t a_addr = smem_u32(A + k * 16384);
                const uint32_t b_addr = smem_u32(B + k * N * 128);
                const uint32_t a_slot = a_tmem0 + (k & 1) * 32;
                if (mode == 2) {
#pragma unroll
                    for (int s = 0; s < 4; ++s) tmem_cp_128x256b(a_slot + s * 8, umma_desc(a_addr + s * 32, 16, 1024));
                }
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint64_t bd = umma_desc(b_addr + s * 32, 16, 1024);
                    const uint32_t acc = (it | k | s) != 0;
                    if (mode >= 3) {
                        const int nacc = mode == 3 ? 2 : 4;
                        const int ai = (k * 4 + s) % nacc;
                        const uint32_t first = it == 0 && k * 4 + s < nacc;
                        mma_tf32(d_tmem + ai * (N * nacc <= 512 ? N : 0), umma_desc(a_addr + s * 32, 16, 1024), bd,
                                 idesc, first ? 0u : 1u);
                    } else if (mode == 0) mma_tf32(d_tmem, umma_desc(a_addr + s * 32, 16, 1024), bd, idesc, acc);
                    else mma_tf32_ts(d_tmem, a_slot + s * 8, bd, idesc, acc);
                }
            }
        }
        mma_commit(&done_bar);
        mbar_wait(&done_bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}


// The product kernel's issue structure: one warp, elect_one() around a K-block
// of 4 back-to-back MMAs (no per-instruction waterfall loop), `nacc`
// independent accumulators in round robin.  cg: 1 (cta_group::1).
template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) probe2_kernel(int kb, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done_bar;
    const int warp = threadIdx.x / 32;
    uint8_t* A = smem;
    uint8_t* B = smem + kb * 16384;
    for (int i = threadIdx.x; i < kb * (16384 + N * 128) / 4; i += blockDim.x)
        reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
    if (warp == 0) tmem_alloc(&tmem_slot, 512);
    if (threadIdx.x == 0) {
        mbar_init(&done_bar, 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc = idesc_tf32(N, false, false);
    if (warp == 1) {
        long long t0 = 0;
        if (elect_one()) t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < kb; ++k) {
                if (elect_one()) {
                    const uint32_t a_addr = smem_u32(A + k * 16384);
                    const uint32_t b_addr = smem_u32(B + k * N * 128);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        const uint32_t acc = (it | k) != 0 || s >= NACC ? 1u : 0u;
                        mma_tf32(tmem + (s % NACC) * N, umma_desc(a_addr + s * 32, 16, 1024),
                                 umma_desc(b_addr + s * 32, 16, 1024), idesc, acc);
                    }
                }
                __syncwarp();
            }
        }
        if (elect_one()) {
            mma_commit(&done_bar);
            mbar_wait(&done_bar, 0);
            cycles[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    }
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}


// probe3: cheap issue.  Descriptors computed once (64-bit base + constant
// start-address steps), GROUP k-blocks (4 * GROUP MMAs) per elect region.
template <int N, int GROUP>
__global__ void __launch_bounds__(128, 1) probe3_kernel(int kb, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t done_bar;
    const int warp = threadIdx.x / 32;
    uint8_t* A = smem;
    uint8_t* B = smem + kb * 16384;
    for (int i = threadIdx.x; i < kb * (16384 + N * 128) / 4; i += blockDim.x)
        reinterpret_cast<float*>(smem)[i] = 0.001f * (i % 97);
    if (warp == 0) tmem_alloc(&tmem_slot, 512);
    if (threadIdx.x == 0) {
        mbar_init(&done_bar, 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc = idesc_tf32(N, false, false);
    if (warp == 1) {
        long long t0 = 0;
        if (elect_one()) t0 = clock64();
        const uint64_t a0 = umma_desc(smem_u32(A), 16, 1024), b0 = umma_desc(smem_u32(B), 16, 1024);
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < kb; k += GROUP) {
                if (elect_one()) {
#pragma unroll
                    for (int g = 0; g < GROUP; ++g) {
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            const uint64_t ad = a0 + static_cast<uint64_t>(((k + g) * 16384 + s * 32) >> 4);
                            const uint64_t bd = b0 + static_cast<uint64_t>(((k + g) * N * 128 + s * 32) >> 4);
                            mma_tf32(tmem, ad, bd, idesc, (it | k | g | s) != 0 ? 1u : 0u);
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (elect_one()) {
            mma_commit(&done_bar);
            mbar_wait(&done_bar, 0);
            cycles[blockIdx.x] = clock64() - t0;
        }
        __syncwarp();
    }
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace

extern "C" int mma_probe(int n, int mode, int kb, int iters, int ctas, unsigned long long* cycles, void* stream) {
    const int smem = 1024 + kb * (16384 + n * 128);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    switch (n) {
        case 64:
            cudaFuncSetAttribute(probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            probe_kernel<64><<<ctas, 128, smem, s>>>(mode, kb, iters, cycles);
            break;
        case 128:
            cudaFuncSetAttribute(probe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            probe_kernel<128><<<ctas, 128, smem, s>>>(mode, kb, iters, cycles);
            break;
        default:
            cudaFuncSetAttribute(probe_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            probe_kernel<256><<<ctas, 128, smem, s>>>(mode, kb, iters, cycles);
    }
    e = cudaGetLastError();
    return static_cast<int>(e);
}

// nacc in {1, 2, 4}; N * nacc <= 512
extern "C" int mma_probe2(int n, int nacc, int kb, int iters, int ctas, unsigned long long* cycles) {
    const int smem = 1024 + kb * (16384 + n * 128);
#define P2(NN, AA)                                                                                   \
    if (n == NN && nacc == AA) {                                                                     \
        cudaFuncSetAttribute(probe2_kernel<NN, AA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        probe2_kernel<NN, AA><<<ctas, 128, smem>>>(kb, iters, cycles);                               \
        return static_cast<int>(cudaGetLastError());                                                 \
    }
    P2(64, 1) P2(64, 2) P2(64, 4) P2(128, 1) P2(128, 2) P2(128, 4) P2(256, 1) P2(256, 2)
#undef P2
    return -1;
}

extern "C" int mma_probe3(int n, int group, int kb, int iters, int ctas, unsigned long long* cycles) {
    const int smem = 1024 + kb * (16384 + n * 128);
#define P3(NN, GG)                                                                                   \
    if (n == NN && group == GG) {                                                                    \
        cudaFuncSetAttribute(probe3_kernel<NN, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        probe3_kernel<NN, GG><<<ctas, 128, smem>>>(kb, iters, cycles);                               \
        return static_cast<int>(cudaGetLastError());                                                 \
    }
    P3(64, 1) P3(64, 2) P3(64, 4) P3(128, 1) P3(128, 2) P3(128, 4) P3(256, 1)
#undef P3
    return -1;
}
