// Non-GEMM kernels of the partitioned step (HBM-bound elementwise /
// row-reduction work).  All launches are asynchronous on the given stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ppb {

constexpr int kMaxTargets = 8;

// Loss head (train_partitioned.cpp:292-315 softmax after the q all-gather,
// :372-416 loss/predictions on rank 0, :432-470 output delta per shard).
//   CE  : in = gathered pre-activation q (rows x F); p = softmax(q);
//         delta_t = p[:, lo_t:hi_t] - onehot;   loss_row = -log(max(p_label,1e-300))
//   MSE : in = gathered output a (rows x F); delta = a - target, masked by a>0
//         when the last layer is relu;          loss_row = sum 0.5 d^2
// prediction: argmax (first max) or a >= 0.5 when F == 1; correct_row = pred == label.
struct LossTargets {
    int n = 0;
    int lo[kMaxTargets] = {};
    int hi[kMaxTargets] = {};
    float* delta[kMaxTargets] = {};  // row 0 of this micro-batch
    long long ld[kMaxTargets] = {};
};

cudaError_t launch_loss_head(const float* in, long long ld_in, int rows, int F, const int* labels,
                             int loss_kind, int relu_last, const LossTargets& t, double* loss_row,
                             int* correct_row, cudaStream_t s);

// Backward merge (train_partitioned.cpp:516-568 / :578-626): sum the
// contributor slots in ascending device order, then the ReLU mask (:564-568).
//   out[r][c] = mask ? (sum_k slot_k[r][c]) * (mask[r][c] > 0) : sum_k slot_k[r][c]
struct ReduceSlots {
    int n = 0;
    const float* slot[kMaxTargets] = {};
};
cudaError_t launch_reduce_mask(const ReduceSlots& slots, long long ld_slot, int rows, int cols,
                               const float* mask, long long ld_mask, float* out, long long ld_out,
                               cudaStream_t s);

// Bias gradient + update (train_partitioned.cpp:507-511 col_sums, :639-649):
// db = column sums of delta (rows x u), bias -= alpha * (db / b).
// Deterministic two-phase reduction over colsum_chunks(rows) row chunks;
// `partial` holds colsum_chunks(rows) x u floats.
constexpr int kColsumChunks = 1024;  // upper bound
inline int colsum_chunks(long long rows) {
    // one block per >= 64 rows, at most 4 blocks per SM
    long long c = (rows + 63) / 64;
    return static_cast<int>(c < 1 ? 1 : (c > 148 * 4 ? 148 * 4 : c));
}
cudaError_t launch_bias_update(const float* delta, long long ld, long long rows, int u, float* partial,
                               float* bias, const double* alpha, float inv_b, cudaStream_t s);
// The first phase alone: colsum_chunks(rows) partial rows of column sums into
// `partial` (per-micro-batch bias gradients, summed later in chunk order).
cudaError_t launch_colsum(const float* delta, long long ld, long long rows, int u, float* partial, cudaStream_t s);

// fp64 (host layout, dense) -> fp32 padded rows.
cudaError_t launch_convert_f64(const double* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s);
cudaError_t launch_convert_f32(const float* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s);

// ---------------------------------------------------------------- conv layers
// Input images: host NHWC rows [b x H*W*C] -> padded NHWC [b][H+2p][W+2p][ld].
cudaError_t launch_pad_input(const double* src64, const float* src32, int imgs, int H, int W, int C, float* dst,
                             int p, long long ld, cudaStream_t s);

// First conv layer with few input channels: im2col rows
// dst[(n*Ho + h)*Wo + w][(r*k + s)*C + c] = x[n][h+r-p][w+s-p][c] (0 outside), pitch ld.
cudaError_t launch_im2col_input(const double* src64, const float* src32, int imgs, int H, int W, int C, int k,
                                int p, float* dst, long long ld, cudaStream_t s);

// Generic conv path: im2col rows of a padded NHWC activation (columns
// (tap, c), zero beyond k*k*C) and the col2im of a partial input gradient into
// a merge slot (channels [c0, c0 + nc)).  See kernels.cu.
cudaError_t launch_im2col_act(const float* x, int imgs, int hp, int wp, long long ldx, int C, int k, int Ho, int Wo,
                              float* dst, long long ldc, cudaStream_t s, int stride = 1);
cudaError_t launch_col2im(const float* dcols, long long ldk, int imgs, int H, int W, int C, int k, int p, int c0,
                          int nc, float* dst, long long ldo, cudaStream_t s, int stride = 1);

// Small-grid conv as a dense layer (kernels.cu: DenseConvGeom): expansion of
// W into Wx, and the fold of dWx + SGD on W + re-expansion.
struct DenseConvGeom {  // see kernels.cu
    int u = 0, C = 0, k = 3, pad = 1, H = 2, W = 2, Ho = 2, Wo = 2;
    long long ldw = 0;   // W row pitch (k*k*ck)
    int ck = 32;
    long long ldx = 0;   // Wx / dWx row pitch (>= Q*C)
};

cudaError_t launch_dense_conv_expand(const DenseConvGeom& g, const float* W, float* Wx, cudaStream_t s);
// bpart / bchunks / bias (optional): the layer's bias update from merge partials, same launch
cudaError_t launch_dense_conv_fold_sgd(const DenseConvGeom& g, const float* dWx, float* W, float* Wx,
                                       const double* alpha, float inv_b, int* flag, cudaStream_t s,
                                       const float* bpart = nullptr, int bchunks = 0, float* bias = nullptr);

cudaError_t launch_spin(long long ns, cudaStream_t s);  // profiling helper

// Layout of a conv layer's output as its consumer reads it.
struct ActLayout {
    int kind = 0;        // 0 padded NHWC [img][hp][wp][ld] at channel col0 + c; 1 CHW-flatten rows [img][ld]
    long long ld = 0;
    int hp = 0, wp = 0, pad = 0;  // kind 0
    int col0 = 0;                 // first channel (shard lo)
};

struct PoolDsts {
    int n = 0;
    float* ptr[kMaxTargets] = {};  // row 0 of this micro-batch in each destination
};

// Max-pool (pool = 2, window 2x2 stride 2, first max wins) or plain relayout
// (pool = 1) of a shard's conv output u: [imgs*Ho*Wo x ldu] into the consumer
// layout on every destination; argmax (0..3 per pooled element) for backward.
cudaError_t launch_pool_fwd(const float* U, long long ldu, int imgs, int Ho, int Wo, int uch, int pool,
                            unsigned char* argmax, const ActLayout& out, const PoolDsts& dsts, cudaStream_t s);

// Backward merge into a conv layer's padded error signal d_pad
// [img][Ho+2q][Wo+2q][ldd] (interior): G = sum of the contributor slots in
// ascending device order (slot layout: 0 pixel-major [img*Hg*Wg x lds] over the
// pooled grid, 1 CHW rows [img][lds]); routed through the pooling argmax;
// masked by the ReLU of the layer's output (mask_kind 1: U rows, 2: the
// padded consumer-layout activation at the same pixel, 3: the pooled
// activation at the window (its max, i.e. U at the argmax), 0: none).
struct ConvMerge {
    ReduceSlots slots;
    int slot_kind = 0;
    long long lds = 0;
    int imgs = 0, Ho = 0, Wo = 0, uch = 0, pool = 1;
    const unsigned char* argmax = nullptr;
    int mask_kind = 0;
    const float* U = nullptr;
    long long ldu = 0;
    const float* act = nullptr;  // padded consumer layout, already offset to this micro-batch
    ActLayout act_layout;
    float* d_pad = nullptr;      // already offset to this micro-batch
    int q = 0;
    long long ldd = 0;
};
// Also writes the merge's bias-gradient partials db_partial[conv_merge_blocks()][uch]
// (column sums of the produced error signal, deterministic per block).
int conv_merge_blocks();
cudaError_t launch_conv_merge(const ConvMerge& m, float* db_partial, cudaStream_t s);

// ---- residual extension (BASELINE configs[3], ResNet-18-style; the
// reference's TinyNet is a chain, tinynet.hpp:50-56, so residual edges are an
// extension of the conv layer description).  A residual layer l adds the
// shortcut of an earlier layer's output a_s to its pre-activation:
//   q_l = conv_l(a_{l-1}) + b_l + shortcut(a_s),
// shortcut = identity, or (ResNet "option A", He et al. 2016 §4.2) the
// positions (f*y, f*x) of a_s with its C_s channels zero-padded to C_l.
struct SkipSrc {
    const float* a = nullptr;  // a_s in its consumer layout (padded NHWC), row 0 of this micro-batch
    ActLayout lay;             // that layout (col0 unused)
    int f = 1;                 // spatial subsampling factor (grid of s / conv grid of l)
    int C = 0;                 // C_s: channels >= C get no shortcut
};
// Forward of a residual and / or average-pooled conv layer's shard: for each
// output position u = U + shortcut (written back into U only for a pooled
// output, where the backward mask needs the pre-activation; otherwise the mask
// reads a = relu(u), since a > 0 <=> u > 0), a = act(u), then a p x p average (pool_avg) or no
// pooling, stored into every destination's consumer layout.  c0 = the
// shard's first channel (absolute).
cudaError_t launch_residual_act(float* U, long long ldu, int imgs, int Ho, int Wo, int uch, int c0, int relu,
                                int pool, const SkipSrc& skip, const ActLayout& out, const PoolDsts& dsts,
                                cudaStream_t s);
// Backward shortcut term for the error signal of a skip-source layer s: the
// error signal of the residual layer l (padded [img][Ho_l+2q][Wo_l+2q][ldd]),
// at channel c + c0 of l's shard for channel c of s's shard.
struct SkipGrad {
    const float* d = nullptr;  // row 0 of this micro-batch
    long long ldd = 0;
    int hq = 0, wq = 0, q = 0;  // padded grid of delta_l
    int f = 1, c0 = 0;
};
// conv_merge for layers the residual extension touches: as launch_conv_merge
// (slot sum in ascending device order, ReLU mask, padded store, bias
// partials) with a p x p average pool routing (pool_avg: every position gets
// G / p^2) and / or the shortcut term added before the mask.  uch % 4 == 0,
// pixel-major slots, mask_kind 1 (U rows: the residual pre-activation) or 2.
cudaError_t launch_conv_merge_res(const ConvMerge& m, int pool_avg, const SkipGrad& sg, float* db_partial,
                                  cudaStream_t s);
// The single-contributor slot of a 3x3 / stride-2 generic conv's dgrad read
// straight from its column-space partial (launch_col2im's arguments, c0 = the
// destination shard's first channel): the merge sums the <= 2 x 2 taps of
// each position (col2im's ascending order, same bits) instead of reading a
// slot col2im wrote.
struct Col2imSrc {
    const float* dcols = nullptr;
    long long ldk = 0;
    int C = 0, p = 0, Ho = 0, Wo = 0, c0 = 0;
};
cudaError_t launch_conv_merge_res_col2im(const ConvMerge& m, int pool_avg, const SkipGrad& sg, const Col2imSrc& cx,
                                         float* db_partial, cudaStream_t s);

// NCCL merge backend: the all-gathered shard outputs [g][rows][u] (rank
// order) into the activation rows [rows][ld] at columns k*u + c.
cudaError_t launch_unpack_gather(const float* recv, int g, int rows, int u, float* dst, long long ld, cudaStream_t s);

// bias -= alpha * (sum_k partial[k][c] / b) over `chunks` partial rows.
cudaError_t launch_bias_from_partials(const float* partial, int chunks, int u, float* bias, const double* alpha,
                                      float inv_b, cudaStream_t s);

// Per-GPU step state, updated once per iteration by the finalize kernel.
struct StepState {
    double alpha;         // alpha_t (train_partitioned.cpp:236, :651)
    double decay;
    int t;                // iterations completed
    int diverged_first;   // 1-based iteration of the first non-finite gradient, 0 if none
    int diverge_flag;     // set by SGD epilogues during the current iteration
    int pad;
};

// Finalize one iteration: history (loss = sum rows / b, ACC = correct / b),
// divergence bookkeeping, alpha *= 1 - decay, t++.
cudaError_t launch_finalize(StepState* st, const double* loss_row, const int* correct_row, int b,
                            double* loss_hist, double* acc_hist, int hist_cap, int write_hist,
                            cudaStream_t s);

}  // namespace ppb
