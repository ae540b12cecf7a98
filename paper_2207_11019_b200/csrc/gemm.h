// Shard GEMM interface shared by the tcgen05 kernel (gemm_tc.cu), the exact
// fp32 SIMT kernel (gemm_simt.cu) and the executor.
//
//   C[m][n] = sum_k A(m,k) * B(n,k)          (fp32 accumulate)
//
// A(m,k) lives at a[m*lda + k] (K-major) or a[k*lda + m] (MN-major); the same
// for B with n in place of m.  The three products of the partitioned step map
// onto it as (reference tinynet.cpp:11-48, train_partitioned.cpp:281,505,515):
//
//   forward  q  = X . W_s^T     A = X  (K-major)  B = W_s (K-major)
//   dgrad    P  = d . W_s       A = d  (K-major)  B = W_s (MN-major)
//   wgrad    dW = d^T . X       A = d  (MN-major) B = X   (MN-major)
//
// The epilogue is where the partitioned step's neighbours are fused: bias +
// activation, the forward all-gather (multi-destination stores into every
// consumer's full-activation buffer), the backward scatter of partial input
// gradients into per-destination slots, the ReLU mask when the reduction is
// trivial, and the SGD update of the weight shard.
#pragma once

#include <cstdint>

namespace ppb {

enum EpiMode : int {
    EPI_STORE = 0,  // out = act(acc + bias[n]) stored to every dst[d]
    EPI_MASK = 1,   // out = acc * (mask[m][mcol0+n] > 0) stored to dst[0]
    EPI_SGD = 2,    // W[m][n] -= alpha * (acc * inv_b); non-finite acc -> *flag = 1
    EPI_SLOTS = 3,  // column segment s of acc stored to seg_dst[s] (backward scatter)
    EPI_MERGE = 4,  // single-contributor conv backward merge (pool argmax + ReLU mask -> padded error)
};

constexpr int kMaxDst = 8;

struct EpiParams {
    int mode = EPI_STORE;
    int M = 0, N = 0;  // valid extent of C
    // EPI_STORE / EPI_MASK: C(m,n) -> dst[d][m*ldd + col0 + n]
    float* dst[kMaxDst] = {};
    int ndst = 0;
    long long ldd = 0;
    int col0 = 0;
    const float* bias = nullptr;  // indexed by n, optional
    int relu = 0;
    // EPI_STORE into a padded NHWC tensor: row m = output pixel (img, h, w) of
    // an ho x wo grid lands at row ((img*hp + h + pad)*wp + w + pad).
    int remap = 0;
    int r_wo = 1, r_howo = 1, r_hp = 1, r_wp = 1, r_pad = 0;
    // EPI_STORE + shortcut of a residual layer (remap only; kernels.h SkipSrc):
    // before the ReLU, C(m, n) += rs_src[((img*rs_hp + f*h + rs_pad)*rs_wp + f*w
    // + rs_pad)*rs_ld + rs_col0 + n] for rs_col0 + n < rs_C (f = rs_f: 1 identity,
    // 2 ResNet option A), (img, h, w) of row m from r_howo / r_wo -- the order
    // ((conv + b) + shortcut) of launch_residual_act in one pass.
    const float* rs_src = nullptr;
    long long rs_ld = 0;
    int rs_hp = 1, rs_wp = 1, rs_pad = 0, rs_col0 = 0, rs_f = 1, rs_C = 0;
    // EPI_STORE + fused 2x2 max-pool (tc kernel; rows = pixels of a
    // pl_ho x pl_wo grid with pl_wo <= 16, so each warp's 32 rows hold whole
    // windows): the window's top-left lane writes the pooled value (first max
    // wins in order (0,0),(0,1),(1,0),(1,1)) to pl_dst[d] in the consumer
    // layout (pl_kind 0: padded NHWC pl_hp x pl_wp, pad pl_pad, pitch pl_ld;
    // 1: CHW-flatten rows of pitch pl_ld) at channel pl_col0 + n, and the
    // window code to pl_arg[pooled pixel * pl_uch + n].
    // pl_on == 3 (grid width 32, TMA-store staging, 128-row tiles of 4 image
    // rows): the windows span the warp pair (q, q^1) holding rows 2y, 2y+1;
    // both stage their chunk in shared memory, meet at a pair barrier and pool
    // from the two boxes (epi_pool_pair).  The pre-pool rows are then not
    // stored at all (nothing else reads them).
    int pl_on = 0;
    int pl_wo = 1, pl_ho = 1;
    float* pl_dst[kMaxDst] = {};
    int pl_ndst = 0;
    int pl_kind = 0;
    long long pl_ld = 0;
    int pl_hp = 1, pl_wp = 1, pl_pad = 0, pl_col0 = 0;
    unsigned char* pl_arg = nullptr;
    int pl_uch = 0;
    // EPI_STORE, segmented columns (dense conv: GEMM column n = (p, c) with
    // p = n / seg_w, c = n % seg_w): C(m, n) -> dst[m*ldd + p*seg_pitch + col0 + c],
    // bias indexed by c.  seg_w is a multiple of 32 (a chunk never straddles).
    int seg_w = 0;
    long long seg_pitch = 0;
    // EPI_MASK
    const float* mask = nullptr;
    long long ldm = 0;
    int mcol0 = 0;
    // EPI_SGD (sgd_t: the product is dW^T, so C(m, n) updates W[n][m])
    float* W = nullptr;
    long long ldw = 0;
    int sgd_t = 0;
    const double* alpha = nullptr;  // device scalar (the reference keeps alpha in double)
    float inv_b = 1.f;
    int* flag = nullptr;
    // EPI_SLOTS: n in [seg_lo[s], seg_hi[s]) -> seg_dst[s][m*seg_ld[s] + n - seg_lo[s]],
    // optionally ReLU-masked by seg_mask[s][m*seg_mask_ld[s] + n] > 0 (used when
    // a layer has a single contributor, so the backward merge is a pure scatter).
    int nseg = 0;
    int seg_lo[kMaxDst] = {};
    int seg_hi[kMaxDst] = {};
    float* seg_dst[kMaxDst] = {};
    long long seg_ld[kMaxDst] = {};
    const float* seg_mask[kMaxDst] = {};
    long long seg_mask_ld[kMaxDst] = {};
    // EPI_MERGE (kernels.h ConvMerge with one contributor, fused): row m = pixel
    // (img, y, x) of the pooled grid mg_hg x mg_wg, column n = channel.  Each
    // pre-pool position (y*pool + dy, x*pool + dx) whose argmax code (dy*2 + dx)
    // matches receives acc (others 0), stored into the padded error signal d.
    // The ReLU mask is read at the POOLED pixel (y, x) of the layer's output
    // activation: the pooled value is the window max, i.e. U at the argmax, so
    // mask(U[argmax] > 0) == mask(pooled > 0).  Positions outside the pooled
    // grid are never written (they stay zero).
    int mg_pool = 1, mg_hg = 1, mg_wg = 1;
    const unsigned char* mg_argmax = nullptr;  // [m][mg_uch]
    int mg_uch = 0;
    const float* mg_mask = nullptr;            // pooled activation [img][mhp][mwp][mld] + mcol0
    long long mg_mld = 0;
    int mg_mhp = 1, mg_mwp = 1, mg_mpad = 0, mg_mcol0 = 0;
    float* mg_d = nullptr;                     // [img][dhp][dwp][dld]
    long long mg_dld = 0;
    int mg_dhp = 1, mg_dwp = 1, mg_dpad = 0;
    // EPI_MERGE with mg_pool == 1, optional: the identity shortcut's gradient
    // for a skip-source layer (kernels.h SkipGrad, f = 1), added before the
    // ReLU mask as conv_merge_res_kernel does: acc += mg_sg[((img*mg_shp + y +
    // mg_spad)*mg_swp + x + mg_spad)*mg_sld + mg_sc0 + n].
    const float* mg_sg = nullptr;
    long long mg_sld = 0;
    int mg_shp = 1, mg_swp = 1, mg_spad = 0, mg_sc0 = 0;
    // EPI_MERGE, optional: column sums of the routed (masked) values, i.e. the
    // bias gradient of the layer below, one row per (CTA, epilogue warp):
    // db_partial[(blockIdx.x * 4 + warp) * N + n], accumulated in shared memory
    // over the CTA's tiles in order (deterministic).  tcgen05 kernels without
    // split-K only; tc_gemm_prepare clears it otherwise.
    float* db_partial = nullptr;
    // timing probes only (wrong results): 2 = skip the epilogue's global stores,
    // 4 = skip the epilogue, 8 = skip the MMAs
    int dbg = 0;
};

// Host-side description of one operand: a row-major fp32 matrix of `rows` x
// `cols` with leading dimension `ld` (elements).  For a K-major operand rows is
// the M (or N) extent and cols is K; for an MN-major operand rows is K.
//
// Implicit-GEMM convolution operands (stride 1, k x k taps) address a padded
// NHWC tensor [img][hp][wp][ch] (or a [u][k*k][ck] weight tensor) through a
// rank-3/4 TMA map instead of a matrix:
//   OP_CONV_ROWS  (A, K-major)  GEMM rows = output pixels; K = (tap, ch block):
//                 box {32 ch, bw, bh, bn} of 128 pixels shifted by the tap
//                 (forward: input x; dgrad: the padded error signal)
//   OP_CONV_KPIX  (A or B, MN-major) K = output pixels (32 per box); MN = channel:
//                 A: the error signal (wgrad); B: the input shifted by the tap of
//                 the 32-column group (tap = col / ck, ch = col % ck)
//   OP_WFLIP      (B, MN-major) dgrad weights: K = (tap, k block), N = input
//                 channel, tap flipped (k*k-1-t), over a [u][k*k][ck] tensor
enum OperandMode : int { OP_DENSE = 0, OP_CONV_ROWS = 1, OP_CONV_KPIX = 2, OP_WFLIP = 3 };

struct ConvGeom {
    int mode = OP_DENSE;
    int wo = 1, howo = 1;    // output pixel grid (rows of the GEMM or its K)
    int bw = 1, bh = 1, bn = 1;  // spatial box (bw*bh*bn = 128 for ROWS, 32 for KPIX)
    int ksz = 1;             // kernel size (taps = ksz*ksz)
    int cblocks = 1;         // 32-channel blocks per tap in the K loop (ROWS, WFLIP)
    int ck = 32;             // per-tap channel pitch of the GEMM N index (KPIX B)
    int off = 0;             // spatial offset into the padded tensor
    int ho = 1;              // output grid rows (howo / wo)
    int krows = 1, kimgs = 1;  // KPIX: rows (howo >= 32) or images (howo < 32) per 32-pixel K block
    int rr = 0;                // ROWS, tc_gemm only: row reuse (box of bh + ksz - 1 rows serves the ksz row taps)
};

struct Operand {
    const float* ptr = nullptr;
    int rows = 0;
    int cols = 0;
    long long ld = 0;
    bool mn_major = false;
    ConvGeom geom;
    // conv tensor extents (elements): [imgs][hp][wp][ch], ch pitch `ld`
    int ch = 0, wp = 0, hp = 0, imgs = 0;
};

// Split-K: the K loop is cut into `splits` ranges of `kps` 32-wide blocks; each
// range's raw partial sums go to ws + split*stride (row pitch ld) and a
// reduction kernel sums the splits in order before the real epilogue.
struct SplitK {
    int splits = 1;
    int kps = 1 << 30;
    float* ws = nullptr;
    long long ld = 0;
    long long stride = 0;
    int trans = 0;  // workspace stored [n][m] (EPI_SGD with sgd_t)
    // optional bias job folded into the reduction launch (wgrad + SGD only):
    // bias[c] -= alpha * inv_b * sum_k bpart[k][c], k in [0, bchunks), c < bu
    const float* bpart = nullptr;
    float* bias = nullptr;
    int bchunks = 0, bu = 0;
    // in-kernel reduction (few splits): each epilogue warp publishes its
    // partial chunks with a per-(tile, CTA, warp slot) counter; the last of
    // the `splits` arrivals sums the splits in order 0..splits-1 and runs the
    // real epilogue (no reduction kernel; counters re-armed to 0)
    int fixup = 0;
    int* counters = nullptr;
    int deferred = 0;  // reduction carried by the next GEMM's SideJob (no kernel here)
    // raw partial sums into workspace slices even when splits == 1 (per
    // micro-batch weight gradients, summed by one reduction after the last)
    int partial = 0;
};

// Padded-position geometry of the halo conv kernel (conv_halo.cu): GEMM row
// p = position in the [imgs][hp][wp] padded grid of the operand A tensor; the
// output pixel (h, w) sits at padded position (h + 1, w + 1); taps (r, s) read
// position p + (r - 1) * wp + (s - 1).
struct HaloGeom {
    int wp = 0, hp = 0;   // padded grid (ho + 2, wo + 2)
    int ho = 0, wo = 0;   // output grid
    int cblocks = 1;      // 32-channel blocks of A
    int rows = 0;         // halo rows staged per CTA: 128 + 2 * (wp + 1)
    long long Mp = 0;     // imgs * hp * wp
    // shared-memory plan (set by halo_conv_prepare)
    int hstages = 3, hstage_bytes = 0;  // halo ring
    int bstages = 0;                    // B ring slots (resident: one per K block)
    int resident = 0;                   // B column slice loaded once per CTA
    int smem = 0;                       // dynamic shared memory bytes
    int dbg = 0;  // timing probes (wrong results): 1 align taps, 2 no epilogue stores, 4 no halo waits
};

// Geometry of the halo weight-gradient kernel (wgrad_halo.cu): K blocks of 32
// output pixels (one image row segment), kbs of them over the batch.
struct WgradGeom {
    int ho = 0, wo = 0;  // output grid (wo % 32 == 0)
    int q = 0;           // ring offset of the error signal's padded layout
    int kbs = 0;         // K blocks (imgs * ho * wo / 32)
};

// A split-K reduction carried by the NEXT GEMM on the stream ("side job"):
// the wgrad + SGD of one layer has no reader before the next step's forward,
// so its reduction (and bias update) runs in the following wgrad GEMM's
// epilogue warps while that GEMM's mainloop occupies the tensor cores,
// instead of as a separate kernel.  Same split order as the reduction kernel
// (sequential 0..splits-1); the bias job sums chunks in 8 lane phases and a
// fixed butterfly.
struct SideJob {
    int on = 0;
    int kind = 0;  // 0: split-K reduction (sk, epi, M, N); 1: dense-conv 2x2 weight update
    int scalar = 0;  // reduction items one at a time (A/B probe)
    int M = 0, N = 0;
    SplitK sk;     // kind 1: only the bias job fields (bpart, bias, bchunks, bu)
    EpiParams epi; // kind 1: alpha, inv_b, flag
    // kind 1 (kernels.h DenseConvGeom for 3x3 / pad 1 / 2x2): dWx -> W, Wx
    const float* dWx = nullptr;
    float* Wm = nullptr;
    float* Wx = nullptr;
    int dc_u = 0, dc_C = 0, dc_ck = 0;
    long long dc_ldw = 0, dc_ldx = 0;
};

struct GemmDesc {
    Operand a, b;
    int M = 0, N = 0, K = 0;
    EpiParams epi;
    // partial_out: store the raw accumulators into split-K workspace slices
    // (ws_alloc provides them) and launch no reduction; `epi` is the epilogue
    // the later reduction (tc_gemm_launch_reduce) applies.  force_splits > 0
    // fixes the split count (every micro-batch's GEMM writes the same slices).
    int partial_out = 0;
    int force_splits = 0;
};

}  // namespace ppb
