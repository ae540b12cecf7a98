/*
 * pipeplan_b200 — C ABI of the B200-native partition-and-merge training step.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `pipeplan` (arXiv 2207.11019 desk-verifier): the layer-wise partitioned
 * forward / merge / backward / SGD step `pipeplan::train_partitioned`, plus
 * the integer planner it consumes.  Every entry point below names the
 * reference interface it replaces (paths relative to the reference's
 * `proj/` directory).  Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions
 *   - Status: every function returns PPB_OK (0) or a PPB_ERR_* code; the
 *     message is in ppb_last_error() (thread-local).  The codes map onto the
 *     reference's exception types so the C++ shim rethrows the same type and
 *     text (std::invalid_argument / std::runtime_error / std::out_of_range).
 *   - Matrices are row-major fp64 on the host, exactly like pipeplan::Matrix
 *     (include/pipeplan/tinynet.hpp:15-27).  On the device the library keeps
 *     fp32 copies; products run on tcgen05 tensor cores in TF32 with fp32
 *     accumulation (PPB_PRECISION_TF32) or on CUDA cores in fp32
 *     (PPB_PRECISION_FP32).
 *   - Device ids inside plans are 1-based as in the reference
 *     (include/pipeplan/model.hpp:32); a context maps plan device k to the
 *     CUDA ordinal device_map[k-1].  Several plan devices may share one GPU.
 *   - Networks are passed as `dims` (L+1 ints: fan_in of layer 1, then each
 *     layer's fan_out — the init_net convention, tinynet.hpp:93-94), `acts`
 *     (L ints, PPB_ACT_*), and all layers' weights / biases concatenated in
 *     layer order (layer l: fan_out x fan_in row-major, then next layer).
 *
 * Flat plan encoding (PartitionPlan, include/pipeplan/partition.hpp:14-47):
 *   [n, Z,
 *    for each sub-module:  index, first_layer, last_layer, D, device_1..device_D,
 *                          for each layer in the span, for each device:
 *                              layer_id, device_id, lo, hi, replicated
 *    boundary_1 .. boundary_{Z-1}    (PPB_BOUNDARY_*)]
 */
#ifndef PIPEPLAN_B200_H
#define PIPEPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ codes */
#define PPB_OK 0
#define PPB_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define PPB_ERR_RUNTIME 2          /* std::runtime_error                     */
#define PPB_ERR_OUT_OF_RANGE 3     /* std::out_of_range                      */
#define PPB_ERR_CUDA 4             /* CUDA failure (runtime_error in the C++ shim) */
#define PPB_ERR_NO_DEVICE 5        /* no CUDA device / extension unusable    */
#define PPB_ERR_BUFFER 6           /* caller buffer too small                */

#define PPB_ACT_IDENTITY 0 /* ActKind::identity     tinynet.hpp:38 */
#define PPB_ACT_RELU 1     /* ActKind::relu                        */
#define PPB_ACT_SOFTMAX 2  /* ActKind::softmax_last                */

#define PPB_LOSS_MSE 0 /* LossKind::mse           tinynet.hpp:39 */
#define PPB_LOSS_CE 1  /* LossKind::cross_entropy                */

#define PPB_BOUNDARY_CONCAT 0 /* BoundaryKind::concat_repartition  partition.hpp:36 */
#define PPB_BOUNDARY_DIRECT 1 /* BoundaryKind::direct                               */

#define PPB_MODE_NONE 0  /* UpdateMode::none (rejected, as in the reference) schedule.hpp:12 */
#define PPB_MODE_SYNC 1  /* UpdateMode::sync_barrier     */
#define PPB_MODE_ASYNC 2 /* UpdateMode::async_per_module */

#define PPB_PRECISION_TF32 0 /* tcgen05 kind::tf32, fp32 accumulate (default) */
#define PPB_PRECISION_FP32 1 /* CUDA-core fp32 FMA chains (tight parity mode)  */

/* Thread-local message of the last failing call ("" if none). */
const char* ppb_last_error(void);

/* Library / device information. */
const char* ppb_version(void);
int ppb_device_count(int* out_count);

/* ------------------------------------------------------------------ planner */

/* split_layer (src/partition.cpp:15-48; partition.hpp:53-56): contiguous
 * output-unit shards of a layer with fan_out units over `n` devices, largest
 * remainder first.  Writes n entries to out_lo/out_hi/out_replicated.
 * Error "layer <id> too narrow to split <n> ways (fan_out <f>)" when
 * fan_out < n and !replicate_narrow. */
int ppb_split_layer(int layer_id, int fan_out, const int* devices, int n, int replicate_narrow,
                    int* out_lo, int* out_hi, int* out_replicated);

/* split_microbatches (src/schedule.cpp:46-55; schedule.hpp:46). */
int ppb_split_microbatches(int b, int m, int* out_sizes);

/* build_plan (src/partition.cpp:110-121): Z spans balanced on fwd_flops over
 * devices 1..n.  fwd_flops may be NULL, meaning the reference's default_costs
 * (2*fan_in*fan_out, src/model.cpp:124-137).  Writes the flat plan; *out_len
 * receives the required length (call with cap=0 to size the buffer). */
int ppb_build_plan(const int* fan_in, const int* fan_out, const double* fwd_flops, int L, int n,
                   int Z, int replicate_narrow, int* out, int cap, int* out_len);

/* build_staged_plan (src/partition.cpp:123-138): one device group per
 * sub-module.  groups = concatenated device ids, group_sizes[Z]. */
int ppb_build_staged_plan(const int* fan_in, const int* fan_out, const double* fwd_flops, int L,
                          const int* groups, const int* group_sizes, int Z, int replicate_narrow,
                          int* out, int cap, int* out_len);

/* build_plan_with_cuts (src/partition.cpp:140-155). */
int ppb_build_plan_with_cuts(const int* fan_in, const int* fan_out, int L, int n,
                             const int* cuts, int ncuts, int replicate_narrow, int* out, int cap,
                             int* out_len);

/* merge_submodules (src/partition.cpp:157-175) on a flat plan, in place
 * (Z is unchanged, so the length is unchanged). */
int ppb_merge_submodules(int* plan, int plan_len, const int* group, int group_len);

/* merge_all (src/partition.cpp:177-182), in place. */
int ppb_merge_all(int* plan, int plan_len);

/* serialize_plan (src/partition.cpp:303-331): the reference's plan JSON,
 * byte-identical to its nlohmann::json dump(2).  provenance: entries joined
 * by '\n' (may be NULL).  *out_len = text length (call with cap = 0 to size;
 * cap must exceed the length for the terminating NUL). */
int ppb_serialize_plan(const int* plan, int plan_len, const char* provenance, char* out, size_t cap,
                       size_t* out_len);

/* parse_plan (src/partition.cpp:333-384) -> flat plan; provenance entries are
 * returned '\n'-joined in `provenance` when non-NULL. */
int ppb_parse_plan(const char* text, int* out, int cap, int* out_len, char* provenance, size_t prov_cap);

/* validate_plan (src/partition.cpp:232-294) against a dense chain. */
int ppb_validate_plan(const int* plan, int plan_len, const int* fan_in, const int* fan_out, int L,
                      int num_cluster_devices /* 0 = no cluster check */);

/* ------------------------------------------------------------------ training */

typedef struct ppb_context ppb_context;
typedef struct ppb_session ppb_session;

/* TrainConfig (include/pipeplan/tinynet.hpp:76-82). */
typedef struct {
    double alpha0;
    double decay;
    int loss; /* PPB_LOSS_* */
    int iterations;
    uint64_t seed;
} ppb_train_config;

/* PartitionedTrainOptions (include/pipeplan/train_partitioned.hpp:9-11) plus
 * the GPU execution knobs. */
typedef struct {
    double receive_timeout_s;  /* watchdog on the step's completion (reference default 30) */
    int precision;             /* PPB_PRECISION_* */
    int multiclass_accuracy;   /* 0: reference behaviour (throw on non-binary labels);
                                  1: extension, ACC = #(pred == label) / b            */
    int use_graph;             /* capture the step in a CUDA graph (1) or launch eagerly (0) */
    int pipeline_gate;         /* F(i,j) waits for B(i,j-gate) (schedule.cpp:293-296); 0 = off */
    int memory_mode;           /* PPB_MEMORY_*: activation stash policy (simulate.hpp:14-16 MemoryMode) */
    int merge_backend;         /* PPB_MERGE_*: transport of the dense layers' merges inside a sub-module */
    int reserved[6];
} ppb_options;

/* Activation stash policy (the reference simulator's MemoryMode,
 * include/pipeplan/simulate.hpp:14-16).  STASH_ALL is the reference
 * executor: every micro-batch's activations stay live until the step's weight
 * gradients, computed once over all b rows (train_partitioned.cpp:228-231,
 * :504-512).  PROPOSED is the paper's schedule: the weight gradient of
 * micro-batch j is accumulated as soon as its backward reaches the layer and
 * its activation / error-signal slots are reused by micro-batch
 * j + min(m, pipeline_gate), so only min(m, gate) micro-batches are resident
 * (tf32 precision; with m = 1 both policies are the same step). */
/* Merge transport (north_star (2)).  P2P: the forward all-gather and the
 * backward reduce-scatter are fused into the producing GEMM epilogues (stores
 * into every consumer GPU's buffers over NVLink; destination sums in
 * ascending device order).  NCCL: dense layers inside a sub-module write
 * their shard locally, ncclAllGather / ncclReduceScatter move it (one
 * communicator per sub-module, libnccl.so.2 loaded at run time) and a kernel
 * lays it out; needs one plan device per GPU and equal shard widths (other
 * layers keep P2P); NCCL's summation order replaces the ascending one. */
#define PPB_MERGE_P2P 0
#define PPB_MERGE_NCCL 1

#define PPB_MEMORY_STASH_ALL 0
#define PPB_MEMORY_PROPOSED 1

/* Layer description for nets with convolution layers (the BASELINE CNN
 * configs; the reference itself is dense-only).  kind = PPB_LAYER_DENSE uses
 * in_units/out_units (fan_in/fan_out) and act only.  kind = PPB_LAYER_CONV:
 * stride-1 ksize x ksize convolution with zero padding `pad` over an input of
 * height x width x in_units (NHWC), activation `act`, then a 2x2 max pool when
 * pool = 2.  The plan shards out_units (channels).  Weights are
 * [out_units][ksize][ksize][in_units] row-major, bias [out_units].  A dense
 * layer after a conv reads the pooled output flattened in (c, h, w) order, so
 * a channel shard is a contiguous feature range; images are passed as
 * [batch][height][width][in_units]. */
#define PPB_LAYER_DENSE 0
#define PPB_LAYER_CONV 1
typedef struct {
    int kind;
    int in_units;
    int out_units;
    int act;
    int height, width;
    int ksize, pad, pool;
    /* residual extension (ResNet-style configs): res_from = 1-based index of
     * an earlier conv layer whose output is added to this conv's
     * pre-activation (identity, or ResNet "option A": every f-th position, C
     * zero-padded, when the grids / widths differ), 0 = none; pool_kind =
     * PPB_POOL_MAX (2x2) or PPB_POOL_AVG (pool x pool average, e.g. a global
     * average pool before the classifier). */
    int res_from;
    int pool_kind;
    int stride; /* conv stride (0 or 1: stride 1; > 1 runs on the generic im2col path) */
} ppb_layer;
#define PPB_POOL_MAX 0
#define PPB_POOL_AVG 1

void ppb_default_options(ppb_options* o);
void ppb_default_config(ppb_train_config* c);

/* A context binds plan devices 1..n_logical to CUDA ordinals. */
int ppb_context_create(const int* device_map, int n_logical, ppb_context** out);
void ppb_context_destroy(ppb_context* ctx);

/* train_partitioned (src/train_partitioned.cpp:121-709;
 * include/pipeplan/train_partitioned.hpp:24-26).  Synchronous: uploads the
 * net and batch, runs cfg->iterations partitioned steps, downloads the trained
 * net (W_out/b_out, same packing as W/b) and the loss / ACC histories
 * (cfg->iterations entries each).  Errors carry the reference's messages
 * ("plan/net shape mismatch: ...", "diverged at iteration t", ...). */
int ppb_train_partitioned(ppb_context* ctx, const int* dims, const int* acts, int L,
                          const double* W, const double* b, const double* X, const int* labels,
                          int batch, const int* plan, int plan_len, int m, int mode,
                          const ppb_train_config* cfg, const ppb_options* opts, double* W_out,
                          double* b_out, double* loss_hist, double* acc_hist);

/* Device bytes the session holds on all its GPUs: total, and the part that
 * scales with the number of resident micro-batches (activations, pre-pool
 * outputs, pool routing, error signals, merge slots, im2col rows). */
int ppb_session_memory(ppb_session* s, size_t* total_bytes, size_t* stash_bytes);

/* Session API: the same step with state resident on the GPUs, for callers
 * that stream batches (and for benchmarking).  A session is
 * train_partitioned() split into its setup / per-iteration / teardown parts;
 * iterating a session k times on one batch is exactly train_partitioned with
 * iterations = k. */
int ppb_session_create(ppb_context* ctx, const int* dims, const int* acts, int L, const double* W,
                       const double* b, int batch, const int* plan, int plan_len, int m, int mode,
                       const ppb_train_config* cfg, const ppb_options* opts, ppb_session** out);
void ppb_session_destroy(ppb_session* s);

/* Same as ppb_session_create / ppb_train_partitioned for nets described by
 * ppb_layer (dense and conv layers). */
int ppb_session_create_layers(ppb_context* ctx, const ppb_layer* layers, int L, const double* W,
                              const double* b, int batch, const int* plan, int plan_len, int m,
                              int mode, const ppb_train_config* cfg, const ppb_options* opts,
                              ppb_session** out);
int ppb_train_partitioned_layers(ppb_context* ctx, const ppb_layer* layers, int L, const double* W,
                                 const double* b, const double* X, const int* labels, int batch,
                                 const int* plan, int plan_len, int m, int mode,
                                 const ppb_train_config* cfg, const ppb_options* opts,
                                 double* W_out, double* b_out, double* loss_hist, double* acc_hist);

/* Upload a batch (host buffers; fp64 as in pipeplan::Batch, or fp32). */
int ppb_session_load_batch(ppb_session* s, const double* X, const int* labels);
int ppb_session_load_batch_f32(ppb_session* s, const float* X, const int* labels);

/* Enqueue `iterations` partitioned steps on the current batch (asynchronous). */
int ppb_session_step(ppb_session* s, int iterations);

/* One end-to-end step for streaming callers: H2D of X/labels from host
 * buffers, the step, and a D2H read of that step's loss (blocking). */
int ppb_session_step_host(ppb_session* s, const float* X, const int* labels, double* loss_out);
/* The same with the reference's fp64 batch rows (Batch::X, tinynet.hpp:58-63). */
int ppb_session_step_host_f64(ppb_session* s, const double* X, const int* labels, double* loss_out);
/* Streaming form: batch t (fp32 X, or fp64 X64 when non-null) is copied into a
 * double-buffered device staging slot on a copy stream while step t-1 still
 * runs; the call returns once step t-1 finished, with its loss in
 * *prev_loss_out (NaN on the first call).  At most two steps in flight; call
 * ppb_session_sync then read the history for the last loss. */
int ppb_session_step_host_pipelined(ppb_session* s, const float* X, const double* X64, const int* labels,
                                    double* prev_loss_out);

/* Block until all enqueued work finished; reports divergence / CUDA errors.
 * Divergence ("diverged at iteration t"): the update is fused into the
 * weight-gradient GEMM epilogue, so the device weights of that step are
 * already updated when the flag is read; the reference throws before its
 * update (train_partitioned.cpp:640-644).  ppb_train_partitioned and the C++
 * drop-in return the same error and no net, as the reference does; only a
 * session caller reading the net after the error sees the difference.  The
 * watchdog deadline is receive_timeout_s per enqueued step (the reference's
 * deadline is per message). */
int ppb_session_sync(ppb_session* s);

/* Histories of all steps taken so far (count = steps); blocking. */
int ppb_session_history(ppb_session* s, double* loss_hist, double* acc_hist, int cap, int* count);

/* Download the current (reassembled) net, same packing as the inputs. */
int ppb_session_get_net(ppb_session* s, double* W_out, double* b_out);

/* Per-layer tensors for parity tests.  kind: 0 = full activation a_l of the
 * current batch (batch x fan_out(l)), 1 = full pre-activation q_L of the last
 * layer (softmax head only), 2 = shard error signal dL/dq_l of plan device
 * `device` (batch x shard units).  layer is 1-based. */
int ppb_session_read_tensor(ppb_session* s, int kind, int layer, int device, double* out,
                            size_t cap_elems, size_t* out_elems);

/* Launch statistics of one step (kernels per step as enqueued). */
int ppb_session_kernels_per_step(ppb_session* s, int* out);

/* Device time (CUDA events on the launching stream, ms) of `iterations`
 * steps on the resident batch; blocking. */
int ppb_session_time_steps(ppb_session* s, int iterations, float* ms_out);

/* Per-op-kind device time: runs `iterations` eager steps with CUDA events
 * around every kernel and accumulates, per kind (0 sync, 1 forward GEMM,
 * 2 dgrad GEMM, 3 wgrad+SGD GEMM, 4 loss head, 5 backward merge, 6 bias
 * update, 7 finalize, 8 peer copy), the milliseconds, launch count and
 * algorithmic FLOPs.  Arrays hold `nkinds` entries. */
int ppb_session_profile(ppb_session* s, int iterations, double* ms, int* count, double* flops,
                        int nkinds);

/* Per-op view of the last ppb_session_profile call: op kind, layer, GEMM
 * tiling (bn | cta_group << 10 | split-K << 12), milliseconds, FLOPs.
 * *count receives the number of ops (call with cap = 0 to size). */
int ppb_session_profile_ops(ppb_session* s, int* kind, int* layer, int* info, double* ms, double* flops, int cap,
                            int* count);

/* Like ppb_session_profile, but the ops overlap as the CUDA graph lets them
 * (every launch is queued behind a spin before the first kernel runs; no
 * per-op serialisation): ppb_session_profile_ops / _starts then give each
 * op's device start and duration on a shared clock (a concurrency timeline,
 * e.g. forward of micro-batch j+1 against backward of micro-batch j). */
int ppb_session_profile_concurrent(ppb_session* s, int iterations);

/* Step structure, same op order as ppb_session_profile_ops: the op's
 * micro-batch (0-based; -1 for once-per-step ops), the plan device of the
 * worker that runs it (1-based; 0 for a GPU's main stream: loss head,
 * hub copies, finalize) and its stream role (0 forward, 1 input gradient /
 * merge, 2 weight gradient / update, 3 main).  The order is the enqueue order
 * of the pipelined schedule (schedule.cpp:254-329). */
int ppb_session_op_meta(ppb_session* s, int* microbatch, int* device, int* role, int cap, int* count);

/* Timeline of the last ppb_session_profile iteration (same op order as
 * ppb_session_profile_ops): start of each op in ms from the first op on its
 * device, and a per-session stream index (eager launch order, not a graph). */
int ppb_session_profile_starts(ppb_session* s, double* start_ms, int* stream_id, int cap, int* count);

/* ------------------------------------------------------------------ diagnostics */

/* One shard GEMM on device pointers (kernel unit tests): C = A.B^T with the
 * operand conventions of csrc/gemm.h and epilogue `mode` (0 store with
 * optional bias/relu, 1 masked store, 2 SGD update of C in place). */
int ppb_debug_gemm(const float* a, int a_rows, int a_cols, long long lda, int a_mn,
                   const float* b, int b_rows, int b_cols, long long ldb, int b_mn, int M, int N,
                   int K, int mode, float* c, long long ldc, const float* bias, int relu,
                   const float* mask, long long ldm, const double* alpha, float inv_b, int* flag,
                   int precision, int force_bn, void* stream);

/* Implicit-GEMM convolution product on device pointers (kernel unit tests):
 * which = 0 forward, 1 dgrad, 2 wgrad; layouts in csrc/conv.h. */
int ppb_debug_conv(int which, const float* x_pad, int N, int H, int W, int C, long long ldx, int pad, int ksz,
                   const float* w, int u, const float* d_pad, long long ldd, float* out, long long ldo,
                   int force_bn, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PIPEPLAN_B200_H */
