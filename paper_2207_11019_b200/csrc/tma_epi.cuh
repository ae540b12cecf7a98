// TMA-store epilogue shared by the tcgen05 kernels (gemm_tc.cu, conv_halo.cu).
//
// The register epilogue stores each accumulator row from its own thread: a
// warp's st.global.v4 touches 32 different rows (16 B each), so a 128 x 256
// tile leaves an SM at a few B/clk and, on single-wave GEMMs, the store tail
// is fully exposed (measured: 18 us of an 85 us 32768 x 256 x 2304 conv GEMM).
// Here each epilogue warp finishes its 32 x 32 chunk in registers (bias,
// ReLU, mask), writes it into a SWIZZLE_128B staging box in shared memory
// (conflict-free: lane = row, 16 B chunk j at j ^ (row & 7)) and one lane
// issues a bulk tensor store per destination; two staging buffers per warp
// let the next chunk's tcgen05.ld overlap the previous store.
//
// Row geometries (TmaStore::rank):
//   2: GEMM row r -> destination row r (plain matrices; the halo kernel's
//      padded-position rows when the destination has the same padded grid)
//   4: GEMM row r = output pixel (img, h, w) of an ho x wo grid -> padded NHWC
//      [img][h + pad][w + pad] (the map's base already points at the interior)
#pragma once

#include <cuda.h>

#include <cstdint>

#include "epilogue.cuh"
#include "gemm.h"
#include "ptx.cuh"

namespace ppb {

constexpr int kEpiWarps = 8;                     // two warps per TMEM lane quarter (alternate column chunks)
constexpr int kEpiStageBytes = kEpiWarps * 4096 + 128;  // one 32 rows x 128 B staging box per epilogue warp + mbarriers
// Double-buffered staging (TmaStore::dbuf): a second set of boxes after the
// mbarrier block (1 KB aligned for SW128), so a warp writes chunk c+1 while
// the bulk store of chunk c is still reading its box (wait_group.read 1).
constexpr int kEpiStage2Off = kEpiWarps * 4096 + 1024;
constexpr int kEpiStageBytesDbuf = kEpiStage2Off + kEpiWarps * 4096;

struct TmaStore {
    CUtensorMap map[kMaxDst];
    int n = 0;     // destinations; 0 = register epilogue
    int rank = 2;  // 2 or 4 (see above)
    int wo = 1, pix = 1;
    int stage_off = 0;  // staging offset (bytes) past the kernel's barrier block
    int tr = 0;         // rank 3 (split-K workspace [split][rows][ld]): 1 = [n][m] (dW^T)
    int segw = 0;       // rank 3 segmented columns (dense conv): box at (n % segw, n / segw, row)
    int pool2 = 0;      // EPI_MERGE through a 2x2 pool: 4 quadrant stores with a stride-2 map
    // ReLU mask of EPI_MERGE (pool 1) / EPI_MASK, same box geometry as the
    // store: TMA-loaded into the staging box (one mbarrier per epilogue warp
    // after the staging boxes), then applied from shared memory
    int mask = 0;
    CUtensorMap mmap;
    int dbuf = 0;  // two staging boxes per warp (plain stores / split-K partials only)
    int mask_pf = 1;  // masked epilogues: issue the first chunk's mask load before the accumulator wait
    // EPI_STORE of a residual layer (identity shortcut): the "mask" box holds
    // the shortcut rows, applied as v = relu(v + box) (tma_store_res_issued)
    int res = 0;
    // EPI_MERGE with a shortcut gradient (EpiParams::mg_sg), halo kernel with
    // two staging boxes per warp: the shortcut-gradient rows are TMA-loaded
    // into the second box next to the mask box (tma_mask_sg_issue)
    int sg = 0;
    CUtensorMap smap;
};

// The staging box of epilogue warp `ewarp` for its `sel`-th buffer.
__device__ __forceinline__ uint8_t* epi_box(uint8_t* stg, int ewarp, int sel) {
    return stg + (sel ? kEpiStage2Off : 0) + ewarp * 4096;
}

// Before rewriting a box: its previous bulk store must have read it.  With
// double buffering the newest group belongs to the other box.
__device__ __forceinline__ void box_wait(int dbuf) {
    if (dbuf) bulk_wait_read<1>();
    else bulk_wait_read<0>();
}

// Host: split-K partial sums through the same staging path: a rank-3 map over
// the workspace ([split][M][ld], or [split][N][ld] transposed).
bool tma_store_setup_splitk(const SplitK& sk, int M, int N, TmaStore* ts);

// Host: encode the destination maps for an epilogue, or leave ts->n = 0 (the
// register epilogue) when the mode / geometry / alignment does not qualify.
// hg != nullptr: the halo kernel (rows are padded positions of hg's grid).
bool tma_store_setup(const EpiParams& e, int M, int N, const HaloGeom* hg, TmaStore* ts);

// Named barrier over the epilogue warps only (id 1).
__device__ __forceinline__ void epi_bar_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
}

// Split-K partial chunk: C(r0 + lane, n .. n + 31) of split `split` into the
// workspace (transposed boxes for the [n][m] layout).
__device__ __forceinline__ void tma_store_partial(const TmaStore& ts, uint8_t* buf, int lane, const float (&v)[32],
                                                  int r0, int n, int split) {
    if (lane == 0) box_wait(ts.dbuf);
    __syncwarp();
    const uint32_t base = smem_u32(buf);
    if (ts.tr) {  // box row = column n + i, 32 consecutive m across the lanes
#pragma unroll
        for (int i = 0; i < 32; ++i)
            st_shared_f32(base + i * 128 + ((((lane >> 2) ^ (i & 7)) << 4) | ((lane & 3) << 2)), v[i]);
    } else {
        const uint32_t row = base + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            st_shared_v4(row + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        if (ts.tr) tma_store_3d(&ts.map[0], buf, r0, n, split);
        else tma_store_3d(&ts.map[0], buf, n, r0, split);
        bulk_commit();
    }
}

__device__ __forceinline__ uint64_t* epi_mask_bar(uint8_t* stage_base, int ewarp) {
    return reinterpret_cast<uint64_t*>(stage_base + kEpiWarps * 4096) + ewarp;
}

// Masked variant: the chunk's ReLU-mask box (the layer's activation at the
// same rows / columns) is TMA-loaded into the staging box, each lane masks
// its row from shared memory (conflict-free, same swizzle), writes the
// result back in place and lane 0 stores it.  v is masked in place (db).
// Issue the ReLU-mask box load of a chunk (the layer's activation at the same
// rows / columns) into the warp's staging box once its previous store has
// read it (lane 0).  Split from tma_store_chunk_masked so an epilogue can
// issue it before waiting for the accumulator and hide its latency.
__device__ __forceinline__ void tma_mask_issue(const TmaStore& ts, uint8_t* buf, uint64_t* bar, int lane, int r0,
                                               int n, bool rank4 = false, int dbuf = 0) {
    if (lane == 0) {
        box_wait(dbuf);  // the previous store from this box has read it
        mbar_arrive_expect_tx(bar, 4096);
        if (ts.rank == 2 && !rank4) {
            tma_load_2d(buf, &ts.mmap, bar, n, r0);
        } else {
            const int img = r0 / ts.pix, rem = r0 - img * ts.pix;
            const int h = rem / ts.wo, w = rem - h * ts.wo;
            tma_load_4d(buf, &ts.mmap, bar, n, w, h, img);
        }
    }
}

// Mask box -> box0 and shortcut-gradient box -> box1 on one mbarrier; box0
// may still be read by this warp's previous bulk store (wait for all).
__device__ __forceinline__ void tma_mask_sg_issue(const TmaStore& ts, uint8_t* box0, uint8_t* box1, uint64_t* bar,
                                                  int lane, int r0, int n) {
    if (lane == 0) {
        box_wait(0);
        mbar_arrive_expect_tx(bar, 8192);
        tma_load_2d(box0, &ts.mmap, bar, n, r0);
        tma_load_2d(box1, &ts.smap, bar, n, r0);
    }
}

// Masked store with the shortcut gradient: v += box1 (shortcut gradient),
// then the ReLU mask from box0, written into box0 and stored (conv_merge_res
// order: sum, shortcut, mask).  v is masked in place (db).
__device__ __forceinline__ void tma_store_masked_sg_issued(const TmaStore& ts, uint8_t* box0, uint8_t* box1,
                                                           uint64_t* bar, uint32_t& phase, int lane, float (&v)[32],
                                                           int r0, int n) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const uint32_t row0 = smem_u32(box0) + lane * 128, row1 = smem_u32(box1) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t off = (j ^ (lane & 7)) << 4;
        float g0, g1, g2, g3, m0, m1, m2, m3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(g0), "=f"(g1), "=f"(g2), "=f"(g3) : "r"(row1 + off));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(m0), "=f"(m1), "=f"(m2), "=f"(m3) : "r"(row0 + off));
        v[4 * j] += g0;
        v[4 * j + 1] += g1;
        v[4 * j + 2] += g2;
        v[4 * j + 3] += g3;
        v[4 * j] = m0 > 0.f ? v[4 * j] : 0.f;
        v[4 * j + 1] = m1 > 0.f ? v[4 * j + 1] : 0.f;
        v[4 * j + 2] = m2 > 0.f ? v[4 * j + 2] : 0.f;
        v[4 * j + 3] = m3 > 0.f ? v[4 * j + 3] : 0.f;
        st_shared_v4(row0 + off, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        for (int d = 0; d < ts.n; ++d) tma_store_2d(&ts.map[d], box0, n, r0);
        bulk_commit();
    }
}

// Second half of the masked store: wait for the issued mask box, mask each
// lane's row from shared memory (conflict-free, same swizzle), write the
// result back in place and lane 0 stores it.  v is masked in place (db).
__device__ __forceinline__ void tma_store_masked_issued(const TmaStore& ts, uint8_t* buf, uint64_t* bar,
                                                        uint32_t& phase, int lane, float (&v)[32], int r0, int n) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t a = row + ((j ^ (lane & 7)) << 4);
        float m0, m1, m2, m3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(m0), "=f"(m1), "=f"(m2), "=f"(m3) : "r"(a));
        v[4 * j] = m0 > 0.f ? v[4 * j] : 0.f;
        v[4 * j + 1] = m1 > 0.f ? v[4 * j + 1] : 0.f;
        v[4 * j + 2] = m2 > 0.f ? v[4 * j + 2] : 0.f;
        v[4 * j + 3] = m3 > 0.f ? v[4 * j + 3] : 0.f;
        st_shared_v4(a, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        if (ts.rank == 2) {
            for (int d = 0; d < ts.n; ++d) tma_store_2d(&ts.map[d], buf, n, r0);
        } else {
            const int img = r0 / ts.pix, rem = r0 - img * ts.pix;
            const int h = rem / ts.wo, w = rem - h * ts.wo;
            for (int d = 0; d < ts.n; ++d) tma_store_4d(&ts.map[d], buf, n, w, h, img);
        }
        bulk_commit();
    }
}

// Residual variant of tma_store_masked_issued (TmaStore::res): v holds conv +
// bias; the issued box holds the shortcut rows; v = act(v + shortcut) in the
// reference order, written back in place and stored.
__device__ __forceinline__ void tma_store_res_issued(const TmaStore& ts, uint8_t* buf, uint64_t* bar, uint32_t& phase,
                                                     int lane, float (&v)[32], int r0, int n, int relu) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t a = row + ((j ^ (lane & 7)) << 4);
        float s0, s1, s2, s3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(s0), "=f"(s1), "=f"(s2), "=f"(s3) : "r"(a));
        v[4 * j] += s0;
        v[4 * j + 1] += s1;
        v[4 * j + 2] += s2;
        v[4 * j + 3] += s3;
        if (relu) {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[4 * j + i] = v[4 * j + i] > 0.f ? v[4 * j + i] : 0.f;
        }
        st_shared_v4(a, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        if (ts.rank == 2) {
            for (int d = 0; d < ts.n; ++d) tma_store_2d(&ts.map[d], buf, n, r0);
        } else {
            const int img = r0 / ts.pix, rem = r0 - img * ts.pix;
            const int h = rem / ts.wo, w = rem - h * ts.wo;
            for (int d = 0; d < ts.n; ++d) tma_store_4d(&ts.map[d], buf, n, w, h, img);
        }
        bulk_commit();
    }
}

// Masked variant of tma_store_chunk: load the mask box, then mask and store.
__device__ __forceinline__ void tma_store_chunk_masked(const TmaStore& ts, uint8_t* buf, uint64_t* bar,
                                                       uint32_t& phase, int lane, float (&v)[32], int r0, int n) {
    tma_mask_issue(ts, buf, bar, lane, r0, n);
    tma_store_masked_issued(ts, buf, bar, phase, lane, v, r0, n);
}

// ReLU mask of the chunk (its rank-4 mask box already issued with
// tma_mask_issue(..., rank4 = true)) applied in registers, no store.
__device__ __forceinline__ void tma_mask_apply_issued(uint8_t* buf, uint64_t* bar, uint32_t& phase, int lane,
                                                      float (&v)[32]) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float m0, m1, m2, m3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(m0), "=f"(m1), "=f"(m2), "=f"(m3)
                     : "r"(row + ((j ^ (lane & 7)) << 4)));
        v[4 * j] = m0 > 0.f ? v[4 * j] : 0.f;
        v[4 * j + 1] = m1 > 0.f ? v[4 * j + 1] : 0.f;
        v[4 * j + 2] = m2 > 0.f ? v[4 * j + 2] : 0.f;
        v[4 * j + 3] = m3 > 0.f ? v[4 * j + 3] : 0.f;
    }
    __syncwarp();
}

// ReLU mask of the chunk (TMA-loaded box) applied in registers, no store.
__device__ __forceinline__ void tma_mask_chunk(const TmaStore& ts, uint8_t* buf, uint64_t* bar, uint32_t& phase,
                                               int lane, float (&v)[32], int r0, int n) {
    tma_mask_issue(ts, buf, bar, lane, r0, n, true);
    tma_mask_apply_issued(buf, bar, phase, lane, v);
}

// Backward merge through a 2x2 max-pool: row r0 + lane = pooled pixel, its 32
// channels route to the argmax position of their window (code byte q =
// dy*2 + dx, zeros elsewhere).  Quadrant q of the 32 pooled pixels is one box
// of a stride-2 tensor map over the error signal's interior, so the four
// quadrants are four bulk stores (staged one after the other).
__device__ __forceinline__ void tma_merge_pool2_chunk(const TmaStore& ts, uint8_t* buf, int lane, const float (&v)[32],
                                                      const uint32_t (&code)[8], int r0, int n) {
    const int img = r0 / ts.pix, rem = r0 - img * ts.pix;
    const int h = rem / ts.wo, w = rem - h * ts.wo;
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * j + k;
                o[k] = ((code[i >> 2] >> (8 * (i & 3))) & 0xffu) == static_cast<uint32_t>(q) ? v[i] : 0.f;
            }
            st_shared_v4(row + ((j ^ (lane & 7)) << 4), o[0], o[1], o[2], o[3]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
            tma_store_4d(&ts.map[0], buf, n, 2 * w + (q & 1), 2 * h + (q >> 1), img);
            bulk_commit();
        }
    }
}

// Registers -> swizzled staging box -> bulk tensor store(s).  All 32 lanes
// call it; lane 0 owns the bulk async-group state.  The warp's next chunk
// (tcgen05.ld, transform) overlaps the store's smem read.
// Stage a 32 x 32 chunk in its SWIZZLE_128B box without storing it (pool
// pair mode: the partner warp reads it).
__device__ __forceinline__ void stage_chunk(uint8_t* buf, int lane, const float (&v)[32]) {
    if (lane == 0) bulk_wait_read<0>();  // a store issued from this box earlier has read it
    __syncwarp();
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_shared_v4(row + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

// Named barrier of the epilogue warp pair (2i, 2i+1), i = (warp - 4) / 2:
// ids 2..5 (0 = __syncthreads, 1 = all epilogue warps).
__device__ __forceinline__ void pair_bar_sync(int epi_warp) {
    asm volatile("bar.sync %0, 64;" ::"r"(2 + (epi_warp >> 1)) : "memory");
}

__device__ __forceinline__ void tma_store_chunk(const TmaStore& ts, uint8_t* buf, int lane, const float (&v)[32],
                                                int r0, int n) {
    if (lane == 0) box_wait(ts.dbuf);  // the previous store from this box has read it
    __syncwarp();
    const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_shared_v4(row + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
        if (ts.segw) {
            for (int d = 0; d < ts.n; ++d) tma_store_3d(&ts.map[d], buf, n % ts.segw, n / ts.segw, r0);
        } else if (ts.rank == 2) {
            for (int d = 0; d < ts.n; ++d) tma_store_2d(&ts.map[d], buf, n, r0);
        } else {
            const int img = r0 / ts.pix, rem = r0 - img * ts.pix;
            const int h = rem / ts.wo, w = rem - h * ts.wo;
            for (int d = 0; d < ts.n; ++d) tma_store_4d(&ts.map[d], buf, n, w, h, img);
        }
        bulk_commit();
    }
}

// The epilogue's value transform without its stores (the TMA path stores).
// EPI_STORE: bias + ReLU.  EPI_MERGE with pool 1 / EPI_MASK: ReLU mask.
// Warp-uniform call (all lanes, any m): the bias row is loaded once per warp
// (lane L holds bias[n0 + L]) and broadcast with shuffles.
__device__ __forceinline__ void epi_values32(const EpiParams& p, int m, int n0, float (&acc)[32], int lane,
                                             bool bias_only = false) {
    if (n0 >= p.N) return;
    if (p.mode == EPI_STORE) {
        if (p.bias != nullptr) {
            const float* b = p.bias + (p.seg_w > 0 ? n0 % p.seg_w : n0);
            if (n0 + 32 <= p.N && (p.seg_w == 0 || n0 % p.seg_w + 32 <= p.seg_w) &&
                (reinterpret_cast<uintptr_t>(b) & 15u) == 0) {
                // the chunk's 32 bias values: warp-uniform float4 loads (L1
                // broadcast), not a load + 32 shuffles per chunk
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(b + i));
                    acc[i] += t.x;
                    acc[i + 1] += t.y;
                    acc[i + 2] += t.z;
                    acc[i + 3] += t.w;
                }
            } else {
                const int bi = p.seg_w > 0 ? (n0 + lane) % p.seg_w : n0 + lane;
                const float bl = n0 + lane < p.N ? __ldg(p.bias + bi) : 0.f;
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] += __shfl_sync(0xffffffffu, bl, i);
            }
        }
        if (m < 0 || m >= p.M || bias_only) return;  // bias_only: shortcut + ReLU in tma_store_res_issued
        // per-lane shortcut rows: staging them through shared memory for
        // coalesced reads measured slower (+95 us on ResNet-18's 64-channel
        // residual layers: the epilogue's shared-memory traffic competes with
        // the MMA operand reads)
        if (p.rs_src != nullptr) epi_residual32(p, m, n0, acc);
        if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = acc[i] > 0.f ? acc[i] : 0.f;
        }
    } else if (m < 0 || m >= p.M) {
        return;
    } else if (p.mode == EPI_MERGE) {
        if (p.mg_sg != nullptr) epi_merge_sg32(p, m, n0, acc);
        if (p.mg_mask != nullptr) {
            const int hw = p.mg_hg * p.mg_wg;
            const int img = m / hw, rem = m - img * hw, y = rem / p.mg_wg, x = rem - y * p.mg_wg;
            const long long mrow = (static_cast<long long>(img) * p.mg_mhp + y + p.mg_mpad) * p.mg_mwp + x + p.mg_mpad;
            const float* mp = p.mg_mask + mrow * p.mg_mld + p.mg_mcol0 + n0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(mp + i));
                acc[i] = t.x > 0.f ? acc[i] : 0.f;
                acc[i + 1] = t.y > 0.f ? acc[i + 1] : 0.f;
                acc[i + 2] = t.z > 0.f ? acc[i + 2] : 0.f;
                acc[i + 3] = t.w > 0.f ? acc[i + 3] : 0.f;
            }
        }
    } else if (p.mode == EPI_MASK) {
        const float* mp = p.mask + static_cast<long long>(m) * p.ldm + p.mcol0 + n0;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(mp + i));
            acc[i] = t.x > 0.f ? acc[i] : 0.f;
            acc[i + 1] = t.y > 0.f ? acc[i + 1] : 0.f;
            acc[i + 2] = t.z > 0.f ? acc[i + 2] : 0.f;
            acc[i + 3] = t.w > 0.f ? acc[i + 3] : 0.f;
        }
    }
}

}  // namespace ppb
