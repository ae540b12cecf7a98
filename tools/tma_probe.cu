// Probe (not part of the product library): TMA box throughput on this B200 --
// does a rank-4 box over a padded NHWC activation ({32 ch, 32 w, rows, 1 img},
// the implicit-conv operand / remapped epilogue store) move bytes as fast as
// a rank-2 box ({32 ch, 128 rows}) of the same size?  One CTA per SM, one
// elected thread issues `iters` 16 KB boxes (loads into a 4-deep smem ring on
// one mbarrier per slot, or bulk stores from smem), over a [imgs][34][34][64]
// fp32 tensor (the VGG conv2 input shape).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -I paper_2207_11019_b200/csrc tools/tma_probe.cu -o tools/_tma_probe.so -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "ptx.cuh"

using namespace ppb;

namespace {

constexpr int kImgs = 512, kHp = 34, kWp = 34, kC = 64;

// mode 0: rank-2 loads, 1: rank-4 loads, 2: rank-2 stores, 3: rank-4 stores
__global__ void __launch_bounds__(128, 1) tma_probe_kernel(const __grid_constant__ CUtensorMap m2,
                                                           const __grid_constant__ CUtensorMap m4, int mode, int iters,
                                                           unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        uint32_t ph[4] = {0u, 0u, 0u, 0u};
        for (int it = 0; it < iters; ++it) {
            const int tile = (blockIdx.x * 977 + it * 148) % (kImgs * 8);  // 128-pixel tiles of interior rows
            const int img = tile / 8, h0 = (tile % 8) * 4;
            const int s = it & 3;
            uint8_t* buf = smem + s * 16384;
            if (mode < 2) {
                if (it >= 4) {  // the previous load into this slot has landed
                    mbar_wait(&bar[s], ph[s]);
                    ph[s] ^= 1u;
                }
                mbar_arrive_expect_tx(&bar[s], 16384);
                if (mode == 0) {
                    // rank-2 view [imgs*hp*wp rows][C]: 128 consecutive padded positions
                    tma_load_2d(buf, &m2, &bar[s], 0, (img * kHp + h0 + 1) * kWp + 1);
                } else {
                    tma_load_4d(buf, &m4, &bar[s], 0, 1, h0 + 1, img);
                }
            } else {
                if (it >= 4) bulk_wait_read<3>();
                if (mode == 2) tma_store_2d(&m2, buf, 0, (img * kHp + h0 + 1) * kWp + 1);
                else tma_store_4d(&m4, buf, 0, 1, h0 + 1, img);
                bulk_commit();
            }
        }
        if (mode < 2) {
            for (int s = 0; s < 4 && s < iters; ++s) mbar_wait(&bar[s], ph[s]);
        } else {
            bulk_wait<0>();
        }
        cycles[blockIdx.x] = clock64() - t0;
    }
}

}  // namespace

extern "C" int tma_probe(float* tensor, int mode, int iters, int ctas, unsigned long long* cycles) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (enc == nullptr) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) return -1;
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    CUtensorMap m2, m4;
    {
        cuuint64_t dims[2] = {kC, static_cast<cuuint64_t>(kImgs) * kHp * kWp};
        cuuint64_t str[1] = {kC * 4};
        cuuint32_t box[2] = {32, 128};
        cuuint32_t es[2] = {1, 1};
        if (enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tensor, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return -2;
    }
    {
        cuuint64_t dims[4] = {kC, kWp, kHp, kImgs};
        cuuint64_t str[3] = {kC * 4, static_cast<cuuint64_t>(kWp) * kC * 4, static_cast<cuuint64_t>(kHp) * kWp * kC * 4};
        cuuint32_t box[4] = {32, 32, 4, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, tensor, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return -3;
    }
    const int smem = 1024 + 4 * 16384;
    cudaFuncSetAttribute(tma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_probe_kernel<<<ctas, 128, smem>>>(m2, m4, mode, iters, cycles);
    return static_cast<int>(cudaGetLastError());
}
