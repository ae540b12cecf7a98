// Diagnostic: TMA load throughput into shared memory as a function of the box
// shape and swizzle mode (no MMA, no compute).  One producer thread per CTA
// keeps `stages` stages of `boxes` boxes in flight; one consumer warp releases
// each stage as soon as it lands.  Used to size the conv/wgrad operand boxes
// (tools/tma_probe.py); not on the training path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "capi_common.h"
#include "gemm_tc.h"
#include "ptx.cuh"

using namespace ppb;

namespace {

__global__ void __launch_bounds__(128, 1) tma_probe_kernel(const __grid_constant__ CUtensorMap map, int rows, int cols,
                                                           int box_rows, int boxes, int stages, int iters) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int box_bytes = box_rows * 128;
    const int stage_bytes = boxes * box_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int nrow_blocks = (rows - box_rows) / box_rows;
    const int ncol_blocks = cols / 32;
    if (warp == 0) {
        if (elect_one()) {
            int st = 0;
            uint32_t ph = 0;
            int cb = 0, rb = static_cast<int>((static_cast<long long>(blockIdx.x) * 997) % nrow_blocks);
            for (int i = 0; i < iters; ++i) {
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], stage_bytes);
                for (int b = 0; b < boxes; ++b) {
                    tma_load_2d(smem + st * stage_bytes + b * box_bytes, &map, &full[st], cb * 32, rb * box_rows);
                    if (++cb == ncol_blocks) {
                        cb = 0;
                        if (++rb == nrow_blocks) rb = 0;
                    }
                }
                if (++st == stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        int st = 0;
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[st], ph);
            __syncwarp();
            if (elect_one()) mbar_arrive(&empty[st]);
            __syncwarp();
            if (++st == stages) {
                st = 0;
                ph ^= 1;
            }
        }
    }
}

}  // namespace

extern "C" int ppb_debug_tma_bw(const float* src, int rows, int cols, int box_rows, int mn_major, int boxes,
                                int stages, int iters, int ctas, void* stream) {
    CUtensorMap map;
    char err[256];
    if (!encode_map(&map, src, rows, cols, cols, box_rows, mn_major != 0, err, sizeof(err))) {
        ppb_set_error(err);
        return PPB_ERR_INVALID_ARGUMENT;
    }
    const int smem = 1024 + stages * boxes * box_rows * 128 + 1024;
    cudaFuncSetAttribute(tma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma_probe_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(map, rows, cols, box_rows, boxes, stages,
                                                                           iters);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        ppb_set_error(cudaGetErrorString(e));
        return PPB_ERR_CUDA;
    }
    return PPB_OK;
}
