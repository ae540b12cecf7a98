// Fused GEMM epilogues (shared by the tcgen05 and SIMT kernels).
//
// One call handles 32 consecutive accumulator columns [n0, n0+32) of row m,
// which is exactly what one tcgen05.ld.32x32b.x32 hands a thread.
#pragma once

#include <cstdint>

#include "gemm.h"

namespace ppb {

__device__ __forceinline__ bool aligned16(const void* p) {
    return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

__device__ __forceinline__ void st_global_v8(float* p, float a, float b, float c, float d, float e, float f, float g,
                                             float h) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d), "f"(e), "f"(f), "f"(g), "f"(h)
                 : "memory");
}

__device__ __forceinline__ void store_row32(float* row, int n0, int nvalid, const float (&v)[32]) {
    // row points at column 0 of the destination row; n0 is a multiple of 32.
    float* p = row + n0;
    if (nvalid >= 32 && (reinterpret_cast<uintptr_t>(p) & 31u) == 0) {
        // 256-bit stores: each lane writes whole 32 B sectors
#pragma unroll
        for (int i = 0; i < 32; i += 8)
            st_global_v8(p + i, v[i], v[i + 1], v[i + 2], v[i + 3], v[i + 4], v[i + 5], v[i + 6], v[i + 7]);
    } else if (nvalid >= 32 && aligned16(p)) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i < nvalid) p[i] = v[i];
        }
    }
}

__device__ __forceinline__ void load_row32(const float* row, int n0, int nvalid, float (&v)[32]) {
    const float* p = row + n0;
    if (nvalid >= 32 && aligned16(p)) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            float4 t = *reinterpret_cast<const float4*>(p + i);
            v[i] = t.x;
            v[i + 1] = t.y;
            v[i + 2] = t.z;
            v[i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = i < nvalid ? p[i] : 0.f;
    }
}

// acc[0..32) += the shortcut of row m (EpiParams::rs_src), m < M.
__device__ __forceinline__ void epi_residual32(const EpiParams& p, int m, int n0, float (&acc)[32]) {
    const int img = m / p.r_howo, rem = m - img * p.r_howo;
    const int h = rem / p.r_wo, w = rem - h * p.r_wo;
    const float* sp = p.rs_src + ((static_cast<long long>(img) * p.rs_hp + h * p.rs_f + p.rs_pad) * p.rs_wp +
                                  w * p.rs_f + p.rs_pad) * p.rs_ld + p.rs_col0 + n0;
    int nv = p.N - n0 < 32 ? p.N - n0 : 32;
    if (p.rs_C - (p.rs_col0 + n0) < nv) nv = p.rs_C - (p.rs_col0 + n0);  // option A: zero-padded channels
    if (nv >= 32 && (reinterpret_cast<uintptr_t>(sp) & 15u) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(sp + i));
            acc[i] += t.x;
            acc[i + 1] += t.y;
            acc[i + 2] += t.z;
            acc[i + 3] += t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < nv) acc[i] += __ldg(sp + i);
    }
}

// acc[0..32) += the shortcut gradient of merge row m (EpiParams::mg_sg),
// 0 <= m < M, columns < N.
__device__ __forceinline__ void epi_merge_sg32(const EpiParams& p, int m, int n0, float (&acc)[32]) {
    const int hw = p.mg_hg * p.mg_wg;
    const int img = m / hw, rem = m - img * hw, y = rem / p.mg_wg, x = rem - y * p.mg_wg;
    const float* sp = p.mg_sg + ((static_cast<long long>(img) * p.mg_shp + y + p.mg_spad) * p.mg_swp + x + p.mg_spad) *
                                    p.mg_sld + p.mg_sc0 + n0;
    if (n0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(sp) & 15u) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(sp + i));
            acc[i] += t.x;
            acc[i + 1] += t.y;
            acc[i + 2] += t.z;
            acc[i + 3] += t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (n0 + i < p.N) acc[i] += __ldg(sp + i);
    }
}

// Apply the epilogue to acc[0..32) = C(m, n0..n0+31).
__device__ __forceinline__ void epilogue32(const EpiParams& p, int m, int n0, float (&acc)[32]) {
    if (m >= p.M || n0 >= p.N) return;
    const int nvalid = p.N - n0 < 32 ? p.N - n0 : 32;
    switch (p.mode) {
        case EPI_STORE: {
            if (p.seg_w > 0) {  // dense conv: chunk n0 lies in segment n0 / seg_w
                const int sp = n0 / p.seg_w, sc = n0 - sp * p.seg_w;
                if (p.bias != nullptr) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] += __ldg(p.bias + sc + i);
                }
                if (p.relu) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = acc[i] > 0.f ? acc[i] : 0.f;
                }
                for (int d = 0; d < p.ndst; ++d)
                    store_row32(p.dst[d] + static_cast<long long>(m) * p.ldd + sp * p.seg_pitch + p.col0 + sc, 0, 32,
                                acc);
                break;
            }
            if (p.bias != nullptr) {
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] += (i < nvalid) ? __ldg(p.bias + n0 + i) : 0.f;
            }
            if (p.rs_src != nullptr) epi_residual32(p, m, n0, acc);
            if (p.relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] = acc[i] > 0.f ? acc[i] : 0.f;
            }
            long long row = m;
            if (p.remap) {
                const int img = m / p.r_howo, rem = m - img * p.r_howo;
                const int h = rem / p.r_wo, w = rem - h * p.r_wo;
                row = (static_cast<long long>(img) * p.r_hp + h + p.r_pad) * p.r_wp + w + p.r_pad;
            }
            for (int d = 0; d < p.ndst; ++d) {
                store_row32(p.dst[d] + row * p.ldd + p.col0, n0, nvalid, acc);
            }
            break;
        }
        case EPI_MASK: {
            float mk[32];
            load_row32(p.mask + static_cast<long long>(m) * p.ldm + p.mcol0, n0, nvalid, mk);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = mk[i] > 0.f ? acc[i] : 0.f;
            store_row32(p.dst[0] + static_cast<long long>(m) * p.ldd + p.col0, n0, nvalid, acc);
            break;
        }
        case EPI_SGD: {
            const float alpha = static_cast<float>(*p.alpha);
            bool bad = false;
            if (p.sgd_t) {  // C = dW^T: lanes hold consecutive m, so W[n][m] stores coalesce across the warp
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    if (i < nvalid) {
                        const float g = acc[i] * p.inv_b;
                        bad |= !isfinite(g);
                        float* wp = p.W + static_cast<long long>(n0 + i) * p.ldw + m;
                        *wp -= alpha * g;
                    }
                }
            } else {
                float w[32];
                float* row = p.W + static_cast<long long>(m) * p.ldw;
                load_row32(row, n0, nvalid, w);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float g = acc[i] * p.inv_b;
                    bad |= (i < nvalid) && !isfinite(g);
                    w[i] -= alpha * g;
                }
                store_row32(row, n0, nvalid, w);
            }
            if (bad && p.flag != nullptr) atomicOr(p.flag, 1);
            break;
        }
        case EPI_SLOTS: {
            for (int s = 0; s < p.nseg; ++s) {
                const int lo = p.seg_lo[s] > n0 ? p.seg_lo[s] : n0;
                const int hi = p.seg_hi[s] < n0 + nvalid ? p.seg_hi[s] : n0 + nvalid;
                if (lo >= hi) continue;
                float v[32];
                if (p.seg_mask[s] != nullptr) {
                    float mk[32];
                    load_row32(p.seg_mask[s] + static_cast<long long>(m) * p.seg_mask_ld[s], n0, nvalid, mk);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = mk[i] > 0.f ? acc[i] : 0.f;
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = acc[i];
                }
                float* row = p.seg_dst[s] + static_cast<long long>(m) * p.seg_ld[s] - p.seg_lo[s];
                if (lo == n0 && hi == n0 + 32) {
                    store_row32(row, n0, 32, v);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int n = n0 + i;
                        if (n >= lo && n < hi) row[n] = v[i];
                    }
                }
            }
            break;
        }
        case EPI_MERGE: {
            const int hw = p.mg_hg * p.mg_wg;
            const int img = m / hw, rem = m - img * hw, y = rem / p.mg_wg, x = rem - y * p.mg_wg;
            uint32_t code[8] = {};
            if (p.mg_pool == 2) {
                const unsigned char* ap = p.mg_argmax + static_cast<long long>(m) * p.mg_uch + n0;
                if ((p.mg_uch & 3) == 0 && nvalid == 32) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) code[i] = __ldg(reinterpret_cast<const uint32_t*>(ap) + i);
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        code[i] = 0;
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            if (4 * i + b < nvalid) code[i] |= static_cast<uint32_t>(__ldg(ap + 4 * i + b)) << (8 * b);
                    }
                }
            }
            if (p.mg_sg != nullptr) epi_merge_sg32(p, m, n0, acc);
            // ReLU mask: the pooled activation (y, x) is the window max = U at the
            // argmax position, so one row of it masks every routed value
            if (p.mg_mask != nullptr) {
                float mk[32];
                const long long mrow = (static_cast<long long>(img) * p.mg_mhp + y + p.mg_mpad) * p.mg_mwp + x + p.mg_mpad;
                load_row32(p.mg_mask + mrow * p.mg_mld + p.mg_mcol0, n0, nvalid, mk);
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[i] = mk[i] > 0.f ? acc[i] : 0.f;
            }
            const int npos = p.mg_pool * p.mg_pool;
            for (int q = 0; q < npos; ++q) {
                const int h = y * p.mg_pool + (q >> 1), w = x * p.mg_pool + (q & 1);
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const bool hit = p.mg_pool == 1 || ((code[i >> 2] >> (8 * (i & 3))) & 0xffu) == static_cast<uint32_t>(q);
                    v[i] = hit ? acc[i] : 0.f;
                }
                const long long drow = (static_cast<long long>(img) * p.mg_dhp + h + p.mg_dpad) * p.mg_dwp + w + p.mg_dpad;
                store_row32(p.mg_d + drow * p.mg_dld, n0, nvalid, v);
            }
            break;
        }
        default:
            break;
    }
}

// Column sums of a warp's 32 x 32 block (row = lane): butterfly transpose-
// reduce, lane L ends with the sum of column L over the 32 rows (fixed order,
// deterministic), added into db_row[n0 + L] (shared memory, this warp only).
__device__ __forceinline__ void db_accumulate(float* db_row, int n0, int N, float (&v)[32], int lane) {
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
        const bool upper = (lane & k) != 0;
#pragma unroll
        for (int i = 0; i < k; ++i) {
            const float send = upper ? v[i] : v[i + k];
            const float keep = upper ? v[i + k] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
        }
    }
    if (n0 + lane < N) db_row[n0 + lane] += v[0];
}

// Fused 2x2 max-pool of a 32 x 32 chunk (EpiParams pl_*): all lanes call it
// with their row's final values (after bias / ReLU); window partners are
// lanes +1, +wo, +wo+1 of the same warp.
__device__ __forceinline__ void epi_pool32(const EpiParams& p, int m, int n0, const float (&v)[32], int lane) {
    const int wo = p.pl_wo, howo = p.pl_wo * p.pl_ho;
    const int img = m / howo, rem = m - img * howo, h = rem / wo, w = rem - h * wo;
    const bool leader = m < p.M && (h & 1) == 0 && (w & 1) == 0;
    float out[32];
    uint32_t code[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const float e1 = __shfl_down_sync(0xffffffffu, v[i], 1);
        const float e2 = __shfl_down_sync(0xffffffffu, v[i], wo);
        const float e3 = __shfl_down_sync(0xffffffffu, v[i], wo + 1);
        float b = v[i];
        uint32_t q = 0;
        if (e1 > b) { b = e1; q = 1; }
        if (e2 > b) { b = e2; q = 2; }
        if (e3 > b) { b = e3; q = 3; }
        out[i] = b;
        code[i >> 2] |= q << (8 * (i & 3));
    }
    if (!leader || n0 >= p.N) return;
    const int nvalid = p.N - n0 < 32 ? p.N - n0 : 32;
    const int Hq = p.pl_ho / 2, Wq = wo / 2, y = h / 2, x = w / 2;
    const long long pp = (static_cast<long long>(img) * Hq + y) * Wq + x;
    unsigned char* ap = p.pl_arg + pp * p.pl_uch + n0;
    if (nvalid == 32 && (p.pl_uch & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(ap)[i] = code[i];
    } else {
        for (int i = 0; i < nvalid; ++i) ap[i] = static_cast<unsigned char>((code[i >> 2] >> (8 * (i & 3))) & 0xffu);
    }
    if (p.pl_kind == 0) {
        const long long o = ((static_cast<long long>(img) * p.pl_hp + y + p.pl_pad) * p.pl_wp + x + p.pl_pad) * p.pl_ld +
                            p.pl_col0;
        for (int d = 0; d < p.pl_ndst; ++d) store_row32(p.pl_dst[d] + o, n0, nvalid, out);
    } else {
        for (int i = 0; i < nvalid; ++i) {
            const long long o = static_cast<long long>(img) * p.pl_ld +
                                static_cast<long long>(p.pl_col0 + n0 + i) * Hq * Wq + static_cast<long long>(y) * Wq + x;
            for (int d = 0; d < p.pl_ndst; ++d) p.pl_dst[d][o] = out[i];
        }
    }
}

// 2x2 max-pool across a warp pair (pl_on == 3, grid width 32): `top` / `bot`
// are the SWIZZLE_128B staging boxes of the warps holding image rows 2y and
// 2y+1 (row r of a box = pixel x = r, 16 B chunk j at j ^ (r & 7)); mtop is
// the top row's first pixel.  Warp `sub` of the pair pools windows
// x = 8*sub .. 8*sub+7; lane = channel, so every pooled pixel is one 128 B
// store per destination and one 32 B argmax store.  Window order and
// tie-breaking as pool_fwd_kernel / epi_pool32: first max wins in
// (0,0), (0,1), (1,0), (1,1).
__device__ __forceinline__ void epi_pool_pair(const EpiParams& p, int mtop, int n0, int lane, uint32_t top,
                                              uint32_t bot, int sub) {
    const int n = n0 + lane;
    if (n >= p.N) return;
    const int wo = p.pl_wo, howo = wo * p.pl_ho;
    const int img = mtop / howo, h = (mtop - img * howo) / wo;
    const int Hq = p.pl_ho >> 1, Wq = wo >> 1, y = h >> 1;
    const uint32_t j = static_cast<uint32_t>(lane) >> 2, kofs = (static_cast<uint32_t>(lane) & 3u) << 2;
    const long long prow = (static_cast<long long>(img) * Hq + y) * Wq;
    const long long obase = (static_cast<long long>(img) * p.pl_hp + y + p.pl_pad) * p.pl_wp + p.pl_pad;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int x = sub * 8 + i;
        const uint32_t r0 = 2u * x, r1 = r0 + 1u;
        const uint32_t o0 = r0 * 128u + ((j ^ (r0 & 7u)) << 4) + kofs;
        const uint32_t o1 = r1 * 128u + ((j ^ (r1 & 7u)) << 4) + kofs;
        float e0, e1, e2, e3;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e0) : "r"(top + o0));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e1) : "r"(top + o1));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e2) : "r"(bot + o0));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e3) : "r"(bot + o1));
        float best = e0;
        unsigned char code = 0;
        if (e1 > best) { best = e1; code = 1; }
        if (e2 > best) { best = e2; code = 2; }
        if (e3 > best) { best = e3; code = 3; }
        p.pl_arg[(prow + x) * p.pl_uch + n] = code;
        const long long o = (obase + x) * p.pl_ld + p.pl_col0 + n;
        for (int d = 0; d < p.pl_ndst; ++d) p.pl_dst[d][o] = best;
    }
}

// Same pool, reading the window partners' rows from the chunk's SWIZZLE_128B
// staging box (row r, 16 B chunk j at j ^ (r & 7)) instead of 96 shuffles:
// only the window leaders load (3 x 8 float4).  The caller has just written
// the box (TMA-store path) and syncs the warp before it is overwritten.
__device__ __forceinline__ void epi_pool32_smem(const EpiParams& p, int m, int n0, const float (&v)[32], int lane,
                                                uint32_t box) {
    const int wo = p.pl_wo, howo = p.pl_wo * p.pl_ho;
    const int img = m / howo, rem = m - img * howo, h = rem / wo, w = rem - h * wo;
    const bool leader = m < p.M && (h & 1) == 0 && (w & 1) == 0 && n0 < p.N;
    if (!leader) return;
    float out[32];
    uint32_t code[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 32; ++i) out[i] = v[i];
    const int rows[3] = {lane + 1, lane + wo, lane + wo + 1};
#pragma unroll
    for (int qq = 0; qq < 3; ++qq) {
        const int r = rows[qq];
        const uint32_t q = static_cast<uint32_t>(qq + 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float e[4];
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(e[0]), "=f"(e[1]), "=f"(e[2]), "=f"(e[3])
                         : "r"(box + r * 128 + ((j ^ (r & 7)) << 4)));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * j + k;
                if (e[k] > out[i]) {
                    out[i] = e[k];
                    code[i >> 2] = (code[i >> 2] & ~(0xffu << (8 * (i & 3)))) | (q << (8 * (i & 3)));
                }
            }
        }
    }
    const int nvalid = p.N - n0 < 32 ? p.N - n0 : 32;
    const int Hq = p.pl_ho / 2, Wq = wo / 2, y = h / 2, x = w / 2;
    const long long pp = (static_cast<long long>(img) * Hq + y) * Wq + x;
    unsigned char* ap = p.pl_arg + pp * p.pl_uch + n0;
    if (nvalid == 32 && (p.pl_uch & 3) == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) reinterpret_cast<uint32_t*>(ap)[i] = code[i];
    } else {
        for (int i = 0; i < nvalid; ++i) ap[i] = static_cast<unsigned char>((code[i >> 2] >> (8 * (i & 3))) & 0xffu);
    }
    if (p.pl_kind == 0) {
        const long long o = ((static_cast<long long>(img) * p.pl_hp + y + p.pl_pad) * p.pl_wp + x + p.pl_pad) * p.pl_ld +
                            p.pl_col0;
        for (int d = 0; d < p.pl_ndst; ++d) store_row32(p.pl_dst[d] + o, n0, nvalid, out);
    } else {
        for (int i = 0; i < nvalid; ++i) {
            const long long o = static_cast<long long>(img) * p.pl_ld +
                                static_cast<long long>(p.pl_col0 + n0 + i) * Hq * Wq + static_cast<long long>(y) * Wq + x;
            for (int d = 0; d < p.pl_ndst; ++d) p.pl_dst[d][o] = out[i];
        }
    }
}

// Row offset (elements) of output row m in the EPI_STORE destination.
__device__ __forceinline__ long long epi_store_row(const EpiParams& p, int m) {
    if (!p.remap) return static_cast<long long>(m) * p.ldd;
    const int img = m / p.r_howo, rem = m - img * p.r_howo;
    const int h = rem / p.r_wo, w = rem - h * p.r_wo;
    return ((static_cast<long long>(img) * p.r_hp + h + p.r_pad) * p.r_wp + w + p.r_pad) * p.ldd;
}

// Element-wise form of the epilogue for the coalesced (row-wise) path: lanes
// of a warp hold consecutive columns n of one row m.  `row_off` is
// epi_store_row(p, m) (EPI_STORE only).  Not used for sgd_t (its natural
// coalescing is along m) or split-K partials (handled by the caller).
__device__ __forceinline__ void epilogue1(const EpiParams& p, int m, int n, float v, long long row_off) {
    if (m >= p.M || n >= p.N) return;
    switch (p.mode) {
        case EPI_STORE: {
            long long col = p.col0 + n;
            int bn = n;
            if (p.seg_w > 0) {
                const int sp = n / p.seg_w;
                bn = n - sp * p.seg_w;
                col = sp * p.seg_pitch + p.col0 + bn;
            }
            if (p.bias != nullptr) v += __ldg(p.bias + bn);
            if (p.relu) v = v > 0.f ? v : 0.f;
            for (int d = 0; d < p.ndst; ++d) p.dst[d][row_off + col] = v;
            break;
        }
        case EPI_MASK: {
            const float mk = p.mask[static_cast<long long>(m) * p.ldm + p.mcol0 + n];
            p.dst[0][static_cast<long long>(m) * p.ldd + p.col0 + n] = mk > 0.f ? v : 0.f;
            break;
        }
        case EPI_SGD: {
            const float g = v * p.inv_b;
            if (!isfinite(g) && p.flag != nullptr) atomicOr(p.flag, 1);
            float* wp = p.W + static_cast<long long>(m) * p.ldw + n;
            *wp -= static_cast<float>(*p.alpha) * g;
            break;
        }
        case EPI_SLOTS: {
            for (int s = 0; s < p.nseg; ++s) {
                if (n < p.seg_lo[s] || n >= p.seg_hi[s]) continue;
                float o = v;
                if (p.seg_mask[s] != nullptr && !(p.seg_mask[s][static_cast<long long>(m) * p.seg_mask_ld[s] + n] > 0.f))
                    o = 0.f;
                p.seg_dst[s][static_cast<long long>(m) * p.seg_ld[s] + n - p.seg_lo[s]] = o;
            }
            break;
        }
        case EPI_MERGE: {
            const int hw = p.mg_hg * p.mg_wg;
            const int img = m / hw, rem = m - img * hw, y = rem / p.mg_wg, x = rem - y * p.mg_wg;
            const int code = p.mg_pool == 2 ? p.mg_argmax[static_cast<long long>(m) * p.mg_uch + n] : 0;
            if (p.mg_sg != nullptr)
                v += p.mg_sg[((static_cast<long long>(img) * p.mg_shp + y + p.mg_spad) * p.mg_swp + x + p.mg_spad) *
                                 p.mg_sld + p.mg_sc0 + n];
            if (p.mg_mask != nullptr) {
                const long long mrow = (static_cast<long long>(img) * p.mg_mhp + y + p.mg_mpad) * p.mg_mwp + x + p.mg_mpad;
                if (!(p.mg_mask[mrow * p.mg_mld + p.mg_mcol0 + n] > 0.f)) v = 0.f;
            }
            const int npos = p.mg_pool * p.mg_pool;
            for (int q = 0; q < npos; ++q) {
                const int h = y * p.mg_pool + (q >> 1), w = x * p.mg_pool + (q & 1);
                const long long drow = (static_cast<long long>(img) * p.mg_dhp + h + p.mg_dpad) * p.mg_dwp + w + p.mg_dpad;
                p.mg_d[drow * p.mg_dld + n] = (p.mg_pool == 1 || code == q) ? v : 0.f;
            }
            break;
        }
        default:
            break;
    }
}

}  // namespace ppb
