// The partitioned training step on B200s: plan -> device-resident shards,
// merge buffers and an event-ordered DAG of kernels per iteration.
//
// Reference: pipeplan::train_partitioned (src/train_partitioned.cpp:121-709).
// One reference worker thread per (sub-module, device) becomes a `Worker`
// with its own forward / backward / update CUDA streams; the Mailbox keys
// (kind, layer, micro-batch, iteration, src) become DAG edges (CUDA events),
// and the value-copy messages become writes into peer-visible merge buffers
// fused into the producing GEMM's epilogue.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gemm_tc.h"
#include "kernels.h"
#include "nccl_merge.h"
#include "planner.h"

namespace ppb {

// One parameterised layer.  Dense layers are the reference's TinyLayer
// (tinynet.hpp:41-48); conv layers extend it (BASELINE.json CNN configs):
// stride-1 k x k convolution with zero padding, activation, optional 2x2 max
// pool, NHWC activations.  The sharded dimension (split_layer's fan_out) is
// out_units: output neurons or output channels.
struct LayerInfo {
    int kind = 0;  // 0 dense, 1 conv
    int in_units = 0, out_units = 0;
    int act = 0;
    int H = 1, W = 1, ksz = 1, pad = 0, pool = 1;  // conv: input grid, kernel, padding, pool factor (1|2)
    // residual extension (kernels.h SkipSrc): q += shortcut(a_res_from) before
    // the activation (1-based layer, 0 = none); pool_avg: p x p average pool
    // (p = pool, e.g. the global 4x4 pool of a ResNet) instead of 2x2 max
    int res_from = 0;
    int pool_avg = 0;
    bool special() const { return res_from > 0 || pool_avg; }  // residual-extension forward / merge kernels
    bool im2col = false;  // first layer with few input channels: explicit im2col rows, dense GEMMs
    // generic conv (grids the 128/32-pixel TMA boxes cannot tile): per-step
    // im2col rows of the padded input, dense GEMMs, col2im of the dgrad partial
    bool generic = false;
    bool dense_delta = false;  // error signal stored unpadded [pixel][ldd] (dense wgrad operand)
    // small grid (H*W <= 4, e.g. VGG's 2x2 layers): the conv as a dense layer
    // over all positions with an expanded weight Wx (kernels.cu DenseConvGeom);
    // input and output stored unpadded NHWC
    bool dense_conv = false;
    int dq() const { return dense_delta ? 0 : ksz - 1 - pad; }  // zero ring of the stored error signal
    int stride = 1;  // conv stride (> 1: the generic im2col path)
    int Ho() const { return (H + 2 * pad - ksz) / stride + 1; }
    int Wo() const { return (W + 2 * pad - ksz) / stride + 1; }
    int Hq() const { return Ho() / pool; }
    int Wq() const { return Wo() / pool; }
    long long in_features() const { return kind ? static_cast<long long>(in_units) * H * W : in_units; }
    long long out_features() const { return kind ? static_cast<long long>(out_units) * Hq() * Wq() : out_units; }
    int host_wcols() const { return kind ? ksz * ksz * in_units : in_units; }
    int ck() const { return (in_units + 31) / 32 * 32; }
    int dev_wcols() const {
        if (!kind) return in_units;
        return im2col || generic ? (ksz * ksz * in_units + 3) / 4 * 4 : ksz * ksz * ck();
    }
};

struct NetDesc {
    std::vector<int> dims;  // L+1 feature counts (dims[0] = input features)
    std::vector<int> acts;  // L (0 identity, 1 relu, 2 softmax_last)
    std::vector<LayerInfo> info;  // L; filled from dims/acts for dense nets
    int L() const { return static_cast<int>(acts.size()); }
};

enum OpKind : int {
    OP_SYNC = 0,
    OP_FWD_GEMM = 1,
    OP_DGRAD_GEMM = 2,
    OP_WGRAD_GEMM = 3,  // wgrad + fused SGD epilogue
    OP_LOSS = 4,
    OP_REDUCE = 5,
    OP_BIAS = 6,
    OP_FINALIZE = 7,
    OP_COPY = 8,
    OP_POOL = 9,        // conv output -> pooled / relaid consumer layout
    OP_CONV_MERGE = 10, // conv backward merge (slots, pool routing, ReLU mask)
    OP_NKINDS = 11,
};

struct SessionConfig {
    double alpha0 = 1e-4;
    double decay = 1e-2;
    int loss = 1;  // 0 mse, 1 cross entropy
    int batch = 0;
    int m = 1;
    int mode = 1;  // 1 sync_barrier, 2 async_per_module
    double timeout_s = 30.0;
    int precision = 0;  // 0 tf32 tcgen05, 1 fp32 SIMT
    int multiclass = 0;
    int use_graph = 1;
    int gate = 2;
    // 0 stash_all (the reference executor: all micro-batches resident, wgrad
    // over all b rows); 1 proposed (ring of min(m, gate) micro-batch slots,
    // weight gradients accumulated per micro-batch)
    int stash = 0;
    // merge transport of the dense layers inside a sub-module: 0 fused
    // epilogue peer stores, 1 NCCL all-gather / reduce-scatter (nccl_merge.h)
    int merge = 0;
};

class Session {
  public:
    Session(const std::vector<int>& device_map, const NetDesc& net, const double* W,
            const double* b, const Plan& plan, const SessionConfig& cfg);
    ~Session();

    void load_batch(const double* X64, const float* X32, const int* labels);
    void step(int iterations);
    void sync();  // throws on divergence / CUDA error / watchdog
    int steps_done() const { return steps_enqueued_; }
    void history(double* loss, double* acc, int cap, int* count);
    void get_net(double* W, double* b);
    size_t read_tensor(int kind, int layer, int device, double* out, size_t cap);
    int kernels_per_step() const { return kernels_per_step_; }
    size_t device_bytes() const;
    size_t stash_bytes() const;
    // device time of `iterations` steps on the launching stream (CUDA events)
    float time_steps(int iterations);
    // one eager iteration per call with per-op CUDA events; accumulates the
    // device time / launch count / algorithmic FLOPs per OpKind
    void profile(int iterations, double* ms, int* count, double* flops, int nkinds);
    // per-op device times of the last profile() call
    int profile_ops(int* kind, int* layer, int* info, double* ms, double* flops, int cap);
    int profile_starts(double* start_ms, int* stream_id, int cap);
    // profile() variant: ops overlap as in the graph (every launch queued
    // behind a spin first), per-op start / end events, no serialisation
    void set_profile_serialised(bool on) { serialise_ = on; }
    // same op order as profile_ops: micro-batch (-1: per-step op), plan
    // device of the worker whose stream runs it (0: a GPU's main stream),
    // stream role (0 forward, 1 input-gradient, 2 weight-gradient, 3 main)
    int op_meta(int* mb, int* device, int* role, int cap);
    double last_loss();
    double step_host(const double* X64, const float* X32, const int* labels);  // load + one step + loss, one sync
    double step_host_pipelined(const double* X64, const float* X32, const int* labels);  // returns step t-1's loss

  private:
    struct Gpu;
    struct Worker;
    struct WLayer;
    struct Op {
        int kind = 0;       // OpKind
        int layer = 0;      // layer the op belongs to (0: none)
        int info = 0;       // GEMM ops: bn | cg << 10 | splits << 12
        double flops = 0;   // algorithmic FLOPs of the op (GEMMs)
        int gpu = 0;
        cudaStream_t stream = nullptr;
        std::function<cudaError_t()> launch;  // may be empty (pure sync node)
        std::vector<int> deps;
        cudaEvent_t ev = nullptr;
        int kernels = 0;
        int mb = -1;        // micro-batch the op belongs to (-1: once per step)
    };

    void build();
    void alloc_buffers();
    void build_ops();
    int add_op(int gpu, cudaStream_t s, std::function<cudaError_t()> f, std::vector<int> deps,
               int kernels, int kind = 0, double flops = 0);
    void enqueue_iteration_timed(std::vector<cudaEvent_t>& t0, std::vector<cudaEvent_t>& t1);
    void enqueue_iteration();
    void capture_graph();
    Gpu& gpu_of(int ordinal);
    float* act_buf(int ordinal, int layer);  // full activation a_layer on that GPU (layer 0 = X)
    long long img_elems(int layer) const;    // floats per sample of act layer `layer` (consumer layout)
    float* q_buf(int ordinal);               // gathered pre-activation of the softmax head
    long long ld_of(int cols) const { return (cols + 3) / 4 * 4; }
    // row offset of micro-batch j in a stash buffer (activation l >= 1, error
    // signal, pre-pool output, ...): its slot in the ring under the proposed
    // memory policy, else its batch offset.  aoff: activation `l` (l = 0 is the
    // batch itself, always resident).
    long long soff(int j) const {
        return ring_ == cfg_.m ? mb_off_[j] : static_cast<long long>(j % ring_) * mb_sizes_[0];
    }
    long long aoff(int l, int j) const { return l == 0 ? mb_off_[j] : soff(j); }
    // residual extension: the layer whose shortcut reads layer s's output (0: none)
    int res_consumer(int s) const {
        for (int l = 1; l <= net_.L(); ++l)
            if (net_.info[l - 1].res_from == s) return l;
        return 0;
    }
    bool skip_source(int s) const { return res_consumer(s) > 0; }
    static bool wgrad_two_streams();
    // NCCL backend: layer l's forward all-gather (and the backward
    // reduce-scatter into it from layer l + 1) go through NCCL
    bool nccl_layer(int l) const;
    int module_index(int l) const;
    void check(cudaError_t e, const char* what);
    void validate_labels(const int* labels) const;

    NetDesc net_;
    Plan plan_;
    SessionConfig cfg_;
    std::vector<int> device_map_;
    std::vector<int> mb_sizes_, mb_off_;
    int ring_ = 1;              // resident micro-batch slots (m under stash_all)
    long long ring_rows_ = 0;   // rows of every stash buffer (b, or ring_ x largest micro-batch)
    bool per_mb_wgrad_ = false; // weight gradients accumulated per micro-batch (proposed)
    std::vector<std::unique_ptr<Gpu>> gpus_;
    std::vector<std::unique_ptr<Worker>> workers_;
    std::vector<std::vector<int>> layer_workers_;  // layer (1-based) -> worker indices (rank order)
    std::vector<Op> ops_;
    int begin_op_ = -1;
    int end_op_ = -1;
    bool fuse_merge_ = true;  // single-contributor conv merges in the dgrad epilogue (PPB_NO_FUSED_MERGE=1 disables)
    int main_gpu_ = 0;  // ordinal holding the loss / history (rank 0 of the last module)
    cudaGraphExec_t graph_exec_ = nullptr;
    cudaGraph_t graph_ = nullptr;
    bool graph_ok_ = false;
    int steps_enqueued_ = 0;
    int hist_cap_ = 0;
    int kernels_per_step_ = 0;
    std::vector<const double*> host_W_, host_b_;
    std::vector<ActLayout> lay_;  // [0..L]: layout of a_l as its consumer reads it
    bool pending_acc_error_ = false;
    int cur_layer_ = 0, cur_info_ = 0, cur_mb_ = -1;
    bool serialise_ = true;
    std::vector<std::unique_ptr<NcclGroup>> nccl_;  // per sub-module (index - 1), NCCL backend only
    std::vector<double> last_op_ms_;
    double* loss_pinned_ = nullptr;  // pinned host slots for step_host's loss read-back
    cudaEvent_t ev_loss_[2] = {nullptr, nullptr};
    int stream_steps_ = 0;
    void stage_batch(const double* X64, const float* X32, const int* labels, int k);
    void convert_staged(int k, bool is64);
    std::vector<double> last_op_start_;  // ms from the first timed op (same device), last profile iteration
};

}  // namespace ppb
