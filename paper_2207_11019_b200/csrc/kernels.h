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
// Deterministic two-phase reduction; `partial` holds kColsumChunks x u floats.
constexpr int kColsumChunks = 32;
cudaError_t launch_bias_update(const float* delta, long long ld, int rows, int u, float* partial,
                               float* bias, const double* alpha, float inv_b, cudaStream_t s);

// fp64 (host layout, dense) -> fp32 padded rows.
cudaError_t launch_convert_f64(const double* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s);
cudaError_t launch_convert_f32(const float* src, int rows, int cols, float* dst, long long ld,
                               cudaStream_t s);

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
