// Partitioned training step executor.  See session.h for the mapping from the
// reference's worker threads / Mailbox to CUDA streams / events, and
// DESIGN.md for buffer layouts and the per-kernel rooflines.
#include "dev_knobs.h"
#include "session.h"

#include "conv.h"
#include "dense_conv.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <set>
#include <stdexcept>
#include <thread>

namespace ppb {

namespace {

std::string S(long long v) { return std::to_string(v); }

[[noreturn]] void cuda_fail(cudaError_t e, const std::string& what) {
    throw std::runtime_error("CUDA error in " + what + ": " + cudaGetErrorString(e));
}

}  // namespace

// ------------------------------------------------------------------ state

struct Session::Gpu {
    int ordinal = 0;
    cudaStream_t main = nullptr;
    StepState* st = nullptr;
    int* labels = nullptr;
    double* loss_row = nullptr;
    int* correct_row = nullptr;
    double* loss_hist = nullptr;
    double* acc_hist = nullptr;
    double* xstage = nullptr;     // staging of the host batch (double-buffered with xstage2)
    double* xstage2 = nullptr;
    int* lstage[2] = {nullptr, nullptr};  // staged labels
    cudaStream_t copy = nullptr;  // host -> device staging stream
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
    std::map<int, float*> act;  // layer -> [b x ld(dims[layer])]
    float* q = nullptr;         // softmax head pre-activation [b x ld(F)]
    std::vector<void*> allocs;
    cudaEvent_t ev_loaded = nullptr;
    cudaEvent_t ev_done = nullptr;
    bool needs_x = false, needs_labels = false;

    size_t bytes_total = 0, bytes_stash = 0;

    // stash: scales with the resident micro-batches (reported by ppb_session_memory)
    void* alloc(size_t bytes, bool stash = false) {
        bytes_total += bytes;
        if (stash) bytes_stash += bytes;
        void* p = nullptr;
        cudaSetDevice(ordinal);
        cudaError_t e = cudaMalloc(&p, bytes < 16 ? 16 : bytes);
        if (e != cudaSuccess) cuda_fail(e, "cudaMalloc(" + S(static_cast<long long>(bytes)) + ")");
        cudaMemset(p, 0, bytes < 16 ? 16 : bytes);
        allocs.push_back(p);
        return p;
    }
};

struct Session::WLayer {
    int layer = 0, lo = 0, hi = 0, u = 0;
    bool replicated = false;
    bool contributor = true;  // writes the layer output / the dgrad partial
    float* W = nullptr;
    long long ldw = 0;
    float* bias = nullptr;
    float* delta = nullptr;  // [b x ldd]
    long long ldd = 0;
    float* partial = nullptr;            // [kColsumChunks x u]
    std::vector<float*> slots;           // per contributor of layer+1 (backward merge inputs)
    long long slot_ld = 0;               // row pitch of the slots
    long long delta_img = 0;             // floats of delta per sample (conv: padded grid)
    float* U = nullptr;                  // conv: pre-pool output of the shard [b*Ho*Wo x ldu]
    bool u_written = true;               // false when the forward epilogue pools across warp pairs
    long long ldu = 0;
    unsigned char* argmax = nullptr;     // conv with pool: [b*Hq*Wq x u]
    float* cols = nullptr;               // generic conv: im2col rows of the input [b*Ho*Wo x ldc]
    long long ldc = 0;
    float* dcols = nullptr;              // generic conv: dgrad partial in column space [b*Ho*Wo x ldk]
    // NCCL merge backend (dense layers): local shard output [rows][u] and the
    // all-gathered [g][rows][u]; this layer's dgrad partial packed per
    // destination rank [g][rows][u_below]; the reduce-scattered sum [rows][u]
    float* ag_send = nullptr;
    float* ag_recv = nullptr;
    float* rs_send = nullptr;
    float* rs_recv = nullptr;
    long long ldk = 0;                   // (dense conv: input-gradient rows [b][H*W*C])
    float* Wx = nullptr;                 // dense conv: expanded weight [Ho*Wo*u x ldwx]
    float* dWx = nullptr;                // dense conv: its gradient
    long long ldwx = 0;
    DenseConvGeom dcg;
    bool merge_fused = false;            // conv: delta written by the dgrad epilogue (EPI_MERGE)
    bool fold_deferred = false;          // dense conv: weight update carried by the next wgrad GEMM
    bool db_colsum = false;              // fused merge without in-epilogue bias partials: column-sum pass
    int db_q = 1;                        // bias partial rows per merge block (dense-conv dgrad: one per position)
    std::vector<std::vector<int>> delta_ready;  // [j] -> op ids that produce delta rows of micro-batch j
    std::vector<int> fwd_op, dgrad_op;   // [j]
    TcGemmPlan p_wgrad;
    GemmDesc d_wgrad;
    // proposed memory policy: per-micro-batch weight-gradient GEMMs writing
    // raw partial sums into slices [j * acc_slices, (j + 1) * acc_slices) of
    // acc_ws, one reduction (+ SGD) after the last micro-batch
    std::vector<TcGemmPlan> p_wg;
    std::vector<GemmDesc> d_wg;
    std::vector<int> wg_op;  // [j]
    TcGemmPlan p_red;
    float* acc_ws = nullptr;
    int acc_slices = 0;
    int cc_mb = 1;  // colsum chunks of one micro-batch's error signal
    std::vector<TcGemmPlan> p_fwd, p_dgrad;
    std::vector<GemmDesc> d_fwd, d_dgrad;
};

struct Session::Worker {
    int module = 0, device = 0, rank = 0, gpu = 0;
    cudaStream_t sf = nullptr, sb = nullptr, su = nullptr;
    cudaStream_t su2 = nullptr;  // second weight-gradient stream (alternate layers; see build_ops)
    std::vector<WLayer> layers;  // span order
    std::vector<int> last_bwd;   // [j] latest backward-side op of this worker
    WLayer& at(int layer) { return layers[layer - layers.front().layer]; }
};

// ------------------------------------------------------------------ helpers

void Session::check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) cuda_fail(e, what);
}

Session::Gpu& Session::gpu_of(int ordinal) {
    for (auto& g : gpus_)
        if (g->ordinal == ordinal) return *g;
    throw std::runtime_error("internal: unknown GPU ordinal " + S(ordinal));
}

float* Session::act_buf(int ordinal, int layer) {
    Gpu& g = gpu_of(ordinal);
    auto it = g.act.find(layer);
    if (it == g.act.end()) throw std::runtime_error("internal: no activation buffer for layer " + S(layer));
    return it->second;
}

float* Session::q_buf(int ordinal) { return gpu_of(ordinal).q; }

// two weight-gradient streams: 2.293 vs 2.317 ms on the VGG-16 step (3 A/B
// pairs on one box); PPB_WGRAD_ONE_STREAM=1 (DEV builds) restores one
bool Session::wgrad_two_streams() { return !dev_knob("PPB_WGRAD_ONE_STREAM"); }

int Session::module_index(int l) const {
    for (const SubModule& sm : plan_.subs)
        if (l >= sm.first_layer && l <= sm.last_layer) return sm.index;
    return 0;
}

bool Session::nccl_layer(int l) const {
    if (cfg_.merge != 1 || l < 1 || l >= net_.L()) return false;
    const LayerInfo& li = net_.info[l - 1];
    const LayerInfo& ln = net_.info[l];
    if (li.kind != 0 || ln.kind != 0 || li.act == 2) return false;
    const int mi = module_index(l);
    if (mi != module_index(l + 1) || mi < 1 || nccl_[mi - 1] == nullptr) return false;
    const auto& ws = layer_workers_[l];
    const int g = static_cast<int>(ws.size());
    if (g < 2 || li.out_units % g != 0 || (li.out_units / g) % 4 != 0) return false;
    for (int wi : ws) {
        const WLayer& wl = workers_[wi]->at(l);
        if (!wl.contributor || wl.replicated || wl.u != li.out_units / g) return false;
        // the backward reduce-scatter pairs contributor k of layer l + 1 with rank k
        const WLayer& wn = workers_[wi]->at(l + 1);
        if (!wn.contributor || wn.replicated) return false;
    }
    return static_cast<int>(layer_workers_[l + 1].size()) == g;
}

size_t Session::device_bytes() const {
    size_t n = 0;
    for (const auto& g : gpus_) n += g->bytes_total;
    return n;
}

size_t Session::stash_bytes() const {
    size_t n = 0;
    for (const auto& g : gpus_) n += g->bytes_stash;
    return n;
}

// ------------------------------------------------------------------ construction

Session::Session(const std::vector<int>& device_map, const NetDesc& net, const double* W,
                 const double* b, const Plan& plan, const SessionConfig& cfg)
    : net_(net), plan_(plan), cfg_(cfg), device_map_(device_map) {
    if (const char* e = getenv("PPB_NO_FUSED_MERGE")) fuse_merge_ = !(*e != '\0' && *e != '0');
    const int L = net_.L();
    // ---- entry validation, in the reference's order (train_partitioned.cpp:124-141)
    if (L < 1) throw std::invalid_argument("net must have at least one layer");
    if (net_.info.empty()) {
        for (int l = 0; l < L; ++l) {
            LayerInfo li;
            li.in_units = net_.dims[l];
            li.out_units = net_.dims[l + 1];
            li.act = net_.acts[l];
            net_.info.push_back(li);
        }
    }
    if (static_cast<int>(net_.info.size()) != L) throw std::invalid_argument("layer description count mismatch");
    net_.dims.assign(1, static_cast<int>(net_.info[0].in_features()));
    for (int l = 0; l < L; ++l) {
        LayerInfo& li = net_.info[l];
        net_.acts[l] = li.act;
        net_.dims.push_back(static_cast<int>(li.out_features()));
        if (li.in_units < 1 || li.out_units < 1)
            throw std::invalid_argument("layer " + S(l + 1) + ": empty weight matrix");
        if (li.kind == 1) {
            if (li.ksz < 1 || li.pad < 0 || li.pool < 1 || (!li.pool_avg && li.pool > 2) || li.stride < 1 ||
                li.Ho() < 1 || li.Wo() < 1 || li.Ho() % li.pool || li.Wo() % li.pool || (l == 0 && li.stride > 1))
                throw std::invalid_argument("layer " + S(l + 1) + ": invalid conv geometry");
            ConvShape cs;
            cs.N = 1;
            cs.H = li.H;
            cs.W = li.W;
            cs.C = li.in_units;
            cs.ksz = li.ksz;
            cs.pad = li.pad;
            cs.u = li.out_units;
            if (!conv_implicit_ok(cs) || li.stride > 1) {
                // generic path: explicit im2col rows + dense GEMMs (layer 1: the
                // staged im2col of X), unpadded error signal
                if (l == 0) li.im2col = true;
                else li.generic = true;
                li.dense_delta = true;
            }
            if (l == L - 1) throw std::invalid_argument("the last layer must be dense (classifier head)");
            if (cfg_.precision == 1)
                throw std::invalid_argument("fp32 precision mode supports dense layers only (conv runs on tcgen05)");
            if (li.act == 2) throw std::invalid_argument("softmax is only valid on the last layer");
        }
        if (l > 0) {
            const LayerInfo& pv = net_.info[l - 1];
            if (li.kind == 1 && pv.kind == 0) throw std::invalid_argument("layer " + S(l + 1) + ": conv after dense");
            if (li.kind == 1 && (li.in_units != pv.out_units || li.H != pv.Hq() || li.W != pv.Wq()))
                throw std::invalid_argument("layers " + S(l) + "," + S(l + 1) + ": shape chain broken");
            if (li.kind == 0 && li.in_units != pv.out_features())
                throw std::invalid_argument("layers " + S(l) + "," + S(l + 1) + ": shape chain broken");
        }
        if (net_.acts[l] == 2 && l != L - 1)
            throw std::invalid_argument("softmax is only valid on the last layer");
        if (li.res_from != 0) {  // residual edge from the output of layer res_from (1-based)
            const int s = li.res_from - 1;
            if (li.kind != 1 || s < 0 || s >= l || net_.info[s].kind != 1)
                throw std::invalid_argument("layer " + S(l + 1) + ": residual source must be an earlier conv layer");
            const LayerInfo& ls = net_.info[s];
            const int f = ls.Hq() / li.Ho();
            if (f < 1 || ls.Hq() != f * li.Ho() || ls.Wq() != f * li.Wo() || li.out_units < ls.out_units)
                throw std::invalid_argument("layer " + S(l + 1) + ": residual shortcut shape mismatch");
            if (li.act == 2) throw std::invalid_argument("layer " + S(l + 1) + ": residual layer with softmax");
        }
        if (li.res_from != 0)
            for (int k = 0; k < l; ++k)
                if (net_.info[k].res_from == li.res_from)
                    throw std::invalid_argument("layer " + S(li.res_from) + ": source of two residual edges");
        if (li.special() && (li.out_units % 4 != 0 || cfg_.precision != 0))
            throw std::invalid_argument("layer " + S(l + 1) + ": residual / average-pool layers need C_out % 4 == 0");
    }
    // few input channels on the first conv: im2col rows (K = k*k*C) instead of
    // 32-channel-padded implicit GEMM taps (K = k*k*32)
    if (net_.info[0].kind == 1 && net_.info[0].in_units < 16) net_.info[0].im2col = true;
    size_t wo = 0, bo = 0;
    for (int l = 0; l < L; ++l) {
        const LayerInfo& li = net_.info[l];
        const size_t nw = static_cast<size_t>(li.out_units) * li.host_wcols();
        for (size_t i = 0; i < nw; ++i)
            if (!std::isfinite(W[wo + i])) throw std::invalid_argument("non-finite weight");
        for (int i = 0; i < li.out_units; ++i)
            if (!std::isfinite(b[bo + i])) throw std::invalid_argument("non-finite bias");
        host_W_.push_back(W + wo);
        host_b_.push_back(b + bo);
        wo += nw;
        bo += li.out_units;
    }
    Chain g;  // the plan shards out_units (neurons or channels) of every layer
    for (int l = 0; l < L; ++l) {
        g.fan_in.push_back(l == 0 ? net_.info[0].in_units : net_.info[l - 1].out_units);
        g.fan_out.push_back(net_.info[l].out_units);
    }
    try {
        validate_plan(plan_, g, 0);
    } catch (const std::exception& e) {
        throw std::runtime_error(std::string("plan/net shape mismatch: ") + e.what());
    }
    if (cfg_.batch < 1) throw std::invalid_argument("batch rows and label count disagree");
    if (cfg_.mode != 1 && cfg_.mode != 2)
        throw std::invalid_argument("train_partitioned needs sync or async update mode");
    mb_sizes_ = split_microbatches(cfg_.batch, cfg_.m);
    mb_off_.assign(cfg_.m + 1, 0);
    for (int j = 0; j < cfg_.m; ++j) mb_off_[j + 1] = mb_off_[j] + mb_sizes_[j];
    // activation stash: every micro-batch resident (stash_all), or a ring of
    // min(m, gate) slots (proposed: F(j) reuses the slots of micro-batch
    // j - ring after its whole backward, weight gradients included)
    if (cfg_.stash == 1 && cfg_.precision != 0)
        throw std::invalid_argument("the proposed memory mode runs on the tf32 tensor-core path");
    per_mb_wgrad_ = cfg_.stash == 1 && cfg_.m > 1;
    ring_ = per_mb_wgrad_ && cfg_.gate > 0 ? std::min(cfg_.m, cfg_.gate) : cfg_.m;
    ring_rows_ = ring_ == cfg_.m ? cfg_.batch : static_cast<long long>(ring_) * mb_sizes_[0];
    if (cfg_.loss == 1 && net_.acts[L - 1] != 2)
        throw std::runtime_error("cross_entropy needs probability outputs (softmax last layer required)");
    if (cfg_.loss == 0 && net_.acts[L - 1] == 2)
        throw std::runtime_error("softmax output requires the cross_entropy loss");
    for (const SubModule& sm : plan_.subs) {
        if (sm.devices.size() > static_cast<size_t>(kMaxDst))
            throw std::invalid_argument("sub-module " + S(sm.index) + " uses more than " + S(kMaxDst) +
                                        " devices (B200 node limit)");
        for (int d : sm.devices)
            if (d < 1 || d > static_cast<int>(device_map_.size()))
                throw std::runtime_error("plan references device " + S(d) + " absent from the context");
    }
    build();
}

Session::~Session() {
    if (loss_pinned_ != nullptr) cudaFreeHost(loss_pinned_);
    for (auto& g : gpus_) {
        cudaSetDevice(g->ordinal);
        cudaDeviceSynchronize();
    }
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (graph_) cudaGraphDestroy(graph_);
    for (auto& op : ops_) {
        if (op.ev) {
            cudaSetDevice(op.gpu);
            cudaEventDestroy(op.ev);
        }
    }
    for (auto& w : workers_) {
        cudaSetDevice(w->gpu);
        cudaStreamDestroy(w->sf);
        cudaStreamDestroy(w->sb);
        cudaStreamDestroy(w->su);
        cudaStreamDestroy(w->su2);
    }
    for (auto& g : gpus_) {
        cudaSetDevice(g->ordinal);
        for (void* p : g->allocs) cudaFree(p);
        if (g->ev_loaded) cudaEventDestroy(g->ev_loaded);
        for (int k = 0; k < 2; ++k) {
            if (g->ev_copied[k]) cudaEventDestroy(g->ev_copied[k]);
            if (g->ev_consumed[k]) cudaEventDestroy(g->ev_consumed[k]);
        }
        if (g->copy) cudaStreamDestroy(g->copy);
        if (g->ev_done) cudaEventDestroy(g->ev_done);
        cudaStreamDestroy(g->main);
    }
}

void Session::build() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        throw std::runtime_error("no CUDA device available for pipeplan_b200");
    }
    // ---- GPUs in first-use order (the plan's device 1 maps to gpus_[0] first)
    std::vector<int> order;
    for (const SubModule& sm : plan_.subs)
        for (int d : sm.devices) {
            const int ord = device_map_[d - 1];
            if (ord < 0 || ord >= ndev) throw std::runtime_error("device map entry " + S(ord) + " is not a CUDA device");
            if (std::find(order.begin(), order.end(), ord) == order.end()) order.push_back(ord);
        }
    for (int ord : order) {
        auto g = std::make_unique<Gpu>();
        g->ordinal = ord;
        check(cudaSetDevice(ord), "cudaSetDevice");
        check(tc_gemm_init_device(), "GEMM attributes");
        check(cudaStreamCreateWithFlags(&g->main, cudaStreamNonBlocking), "stream");
        check(cudaEventCreateWithFlags(&g->ev_loaded, cudaEventDisableTiming), "event");
        check(cudaStreamCreateWithFlags(&g->copy, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < 2; ++k) {
            check(cudaEventCreateWithFlags(&g->ev_copied[k], cudaEventDisableTiming), "event");
            check(cudaEventCreateWithFlags(&g->ev_consumed[k], cudaEventDisableTiming), "event");
        }
        check(cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming), "event");
        gpus_.push_back(std::move(g));
    }
    // peer access between every pair of distinct GPUs (NVLink / NVSwitch)
    for (auto& a : gpus_)
        for (auto& c : gpus_) {
            if (a->ordinal == c->ordinal) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, a->ordinal, c->ordinal);
            if (!can) throw std::runtime_error("GPU " + S(a->ordinal) + " cannot access peer GPU " + S(c->ordinal));
            cudaSetDevice(a->ordinal);
            cudaError_t e = cudaDeviceEnablePeerAccess(c->ordinal, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_fail(e, "peer access");
            cudaGetLastError();
        }
    // ---- workers, one per (sub-module, device) as in train_partitioned.cpp:150-176
    const int L = net_.L();
    layer_workers_.assign(L + 1, {});
    for (const SubModule& sm : plan_.subs) {
        for (size_t r = 0; r < sm.devices.size(); ++r) {
            auto w = std::make_unique<Worker>();
            w->module = sm.index;
            w->device = sm.devices[r];
            w->rank = static_cast<int>(r);
            w->gpu = device_map_[w->device - 1];
            check(cudaSetDevice(w->gpu), "cudaSetDevice");
            // the forward / input-gradient chain is the critical path: its streams get
            // the highest priority, the weight-gradient stream (fills the gaps) the lowest
            int prio_lo = 0, prio_hi = 0;
            cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
            static const bool no_prio = dev_knob("PPB_NO_PRIO");
            if (no_prio) prio_lo = prio_hi = 0;
            check(cudaStreamCreateWithPriority(&w->sf, cudaStreamNonBlocking, prio_hi), "stream");
            check(cudaStreamCreateWithPriority(&w->sb, cudaStreamNonBlocking, prio_hi), "stream");
            check(cudaStreamCreateWithPriority(&w->su, cudaStreamNonBlocking, prio_lo), "stream");
            check(cudaStreamCreateWithPriority(&w->su2, cudaStreamNonBlocking, prio_lo), "stream");
            for (int l = sm.first_layer; l <= sm.last_layer; ++l) {
                const Shard& s = sm.layer_shards(l)[r];
                WLayer wl;
                wl.layer = l;
                wl.lo = s.lo;
                wl.hi = s.hi;
                wl.u = s.hi - s.lo;
                wl.replicated = s.replicated;
                wl.contributor = !s.replicated || r == 0;  // train_partitioned.cpp:181-190
                w->layers.push_back(std::move(wl));
                layer_workers_[l].push_back(static_cast<int>(workers_.size()));
            }
            w->last_bwd.assign(cfg_.m, -1);
            workers_.push_back(std::move(w));
        }
    }
    // loss / history live with rank 0 of the last module (train_partitioned.cpp:372)
    main_gpu_ = workers_[layer_workers_[L].front()]->gpu;
    // NCCL merge backend: one communicator per multi-device sub-module
    // (rank = position in its device list)
    nccl_.clear();
    nccl_.resize(plan_.subs.size());
    if (cfg_.merge == 1) {
        if (cfg_.precision != 0) throw std::invalid_argument("the NCCL merge backend runs on the tf32 path");
        for (const SubModule& sm : plan_.subs) {
            if (sm.devices.size() < 2) continue;
            std::vector<int> ords;
            for (int d : sm.devices) ords.push_back(device_map_[d - 1]);
            nccl_[sm.index - 1] = nccl_group_create(ords);
        }
    }
    alloc_buffers();
    build_ops();
    if (cfg_.use_graph) capture_graph();
}

long long Session::img_elems(int layer) const {
    const ActLayout& a = lay_[layer];
    return a.kind == 1 ? a.ld : static_cast<long long>(a.hp) * a.wp * a.ld;
}

void Session::alloc_buffers() {
    const int L = net_.L();
    const int b = cfg_.batch;
    const int F = net_.dims[L];
    const bool softmax = net_.acts[L - 1] == 2;
    hist_cap_ = 1 << 16;
    // dense conv for small grids (fewer MACs than the 3x3 implicit GEMM): every
    // shard width a multiple of 32 (segmented epilogue chunks), C % 4 == 0
    // (unpadded input rows are the K dimension); its output must feed a pool /
    // dense consumer or another dense-conv layer.  Decided from the top down.
    {
        static const bool off = dev_knob("PPB_NO_DENSE_CONV");
        for (int i = L - 1; i >= 1 && !off; --i) {
            LayerInfo& li = net_.info[i];
            if (li.kind != 1 || li.generic || li.im2col || li.H * li.W > 4 || li.in_units % 4 != 0 ||
                li.ksz * li.ksz > 25 || cfg_.precision != 0 || li.special() || skip_source(i + 1) || li.stride > 1)
                continue;
            bool ok = true;
            for (int wi : layer_workers_[i + 1]) ok = ok && workers_[wi]->at(i + 1).u % 32 == 0;
            const LayerInfo* nx = i + 1 < L ? &net_.info[i + 1] : nullptr;
            if (li.pool == 1 && nx != nullptr && nx->kind == 1 && !nx->dense_conv) ok = false;
            if (ok) {
                li.dense_conv = true;
                li.dense_delta = true;
            }
        }
    }
    // layout of a_l as layer l+1 reads it: padded NHWC for a conv consumer,
    // dense rows (CHW flatten after a conv) for a dense consumer
    lay_.assign(L + 1, ActLayout{});
    for (int l = 0; l <= L; ++l) {
        ActLayout& a = lay_[l];
        if (l == 0 && net_.info[0].im2col) {
            const LayerInfo& c = net_.info[0];
            a.kind = 2;  // im2col rows [pixel][k*k*C]
            a.hp = c.Ho() * c.Wo();
            a.wp = 1;
            a.ld = (c.ksz * c.ksz * c.in_units + 31) / 32 * 32;  // 128 B rows: whole-line TMA fetches
        } else if (l < L && net_.info[l].kind == 1) {
            const LayerInfo& c = net_.info[l];
            a.kind = 0;
            a.pad = c.dense_conv ? 0 : c.pad;  // dense conv reads unpadded rows [img][(q, c)]
            a.hp = c.H + 2 * a.pad;
            a.wp = c.W + 2 * a.pad;
            a.ld = ld_of(c.in_units);
        } else {
            a.kind = 1;
            a.ld = ld_of(net_.dims[l]);
        }
    }
    // which GPUs need which full activations
    std::map<int, std::set<int>> need;  // layer -> ordinals
    for (int wi : layer_workers_[1]) need[0].insert(workers_[wi]->gpu);
    for (int l = 1; l < L; ++l) {
        for (int wi : layer_workers_[l]) need[l].insert(workers_[wi]->gpu);
        for (int wi : layer_workers_[l + 1]) need[l].insert(workers_[wi]->gpu);
    }
    if (!softmax)
        for (int wi : layer_workers_[L]) need[L].insert(workers_[wi]->gpu);
    // a residual layer reads the shortcut source's full activation on its GPU
    for (int l = 1; l <= L; ++l)
        if (net_.info[l - 1].res_from > 0)
            for (int wi : layer_workers_[l]) need[net_.info[l - 1].res_from].insert(workers_[wi]->gpu);
    for (auto& [l, set] : need)
        for (int ord : set) {
            Gpu& g = gpu_of(ord);
            const long long rows = l == 0 ? b : ring_rows_;  // the batch X stays resident
            g.act[l] = static_cast<float*>(g.alloc(sizeof(float) * rows * img_elems(l), l > 0));
        }
    for (int wi : layer_workers_[1]) gpu_of(workers_[wi]->gpu).needs_x = true;
    for (int wi : layer_workers_[L]) {
        Gpu& g = gpu_of(workers_[wi]->gpu);
        g.needs_labels = true;
        if (softmax && g.q == nullptr) g.q = static_cast<float*>(g.alloc(sizeof(float) * ring_rows_ * ld_of(F), true));
    }
    for (auto& gp : gpus_) {
        Gpu& g = *gp;
        g.st = static_cast<StepState*>(g.alloc(sizeof(StepState)));
        StepState init{cfg_.alpha0, cfg_.decay, 0, 0, 0, 0};
        check(cudaMemcpy(g.st, &init, sizeof(init), cudaMemcpyHostToDevice), "init state");
        g.labels = static_cast<int*>(g.alloc(sizeof(int) * b));
        g.loss_row = static_cast<double*>(g.alloc(sizeof(double) * b));
        g.correct_row = static_cast<int*>(g.alloc(sizeof(int) * b));
        if (g.ordinal == main_gpu_) {
            g.loss_hist = static_cast<double*>(g.alloc(sizeof(double) * hist_cap_));
            g.acc_hist = static_cast<double*>(g.alloc(sizeof(double) * hist_cap_));
        }
        if (g.needs_x) {
            g.xstage = static_cast<double*>(g.alloc(sizeof(double) * b * net_.dims[0]));
            g.xstage2 = static_cast<double*>(g.alloc(sizeof(double) * b * net_.dims[0]));
        }
        for (int k = 0; k < 2; ++k) g.lstage[k] = static_cast<int*>(g.alloc(sizeof(int) * b));
    }
    // shard weights, bias, error signals (+ conv pre-pool outputs / argmax)
    std::vector<float> tmp;
    for (auto& wp : workers_) {
        Worker& w = *wp;
        Gpu& g = gpu_of(w.gpu);
        for (WLayer& wl : w.layers) {
            const LayerInfo& li = net_.info[wl.layer - 1];
            if ((li.special() || skip_source(wl.layer)) && wl.u % 4 != 0)
                throw std::invalid_argument("layer " + S(wl.layer) + ": residual-extension shards need a multiple of 4 "
                                            "channels (shard of " + S(wl.u) + ")");
            const int hc = li.host_wcols();
            wl.ldw = li.kind ? li.dev_wcols() : ld_of(li.in_units);
            wl.W = static_cast<float*>(g.alloc(sizeof(float) * wl.u * wl.ldw));
            wl.bias = static_cast<float*>(g.alloc(sizeof(float) * wl.u));
            wl.ldd = ld_of(wl.u);
            if (li.kind == 1) {
                const int q = li.dq();
                wl.delta_img = static_cast<long long>(li.Ho() + 2 * q) * (li.Wo() + 2 * q) * wl.ldd;
                const bool consumer_dense = wl.layer < L && net_.info[wl.layer].kind == 0;
                if (li.pool == 2 || consumer_dense || li.special()) {
                    wl.ldu = ld_of(wl.u);
                    wl.U = static_cast<float*>(g.alloc(sizeof(float) * ring_rows_ * li.Ho() * li.Wo() * wl.ldu, true));
                }
                if (li.pool == 2 && !li.pool_avg)
                    wl.argmax = static_cast<unsigned char*>(
                        g.alloc(static_cast<size_t>(ring_rows_) * li.Hq() * li.Wq() * wl.u, true));
                if (li.dense_conv) {
                    const int P = li.Ho() * li.Wo(), Q = li.H * li.W;
                    wl.ldwx = static_cast<long long>(Q) * li.in_units;
                    wl.Wx = static_cast<float*>(g.alloc(sizeof(float) * P * wl.u * wl.ldwx));
                    wl.dWx = static_cast<float*>(g.alloc(sizeof(float) * P * wl.u * wl.ldwx));
                    wl.ldk = wl.ldwx;
                    wl.dcols = static_cast<float*>(g.alloc(sizeof(float) * ring_rows_ * wl.ldk, true));
                    DenseConvGeom& dg = wl.dcg;
                    dg.u = wl.u;
                    dg.C = li.in_units;
                    dg.k = li.ksz;
                    dg.pad = li.pad;
                    dg.H = li.H;
                    dg.W = li.W;
                    dg.Ho = li.Ho();
                    dg.Wo = li.Wo();
                    dg.ck = li.ck();
                    dg.ldx = wl.ldwx;
                }
                if (li.generic) {
                    const long long pix = ring_rows_ * li.Ho() * li.Wo();
                    const int kc = li.ksz * li.ksz * li.in_units;
                    wl.ldc = (kc + 31) / 32 * 32;
                    wl.ldk = ld_of(kc);
                    wl.cols = static_cast<float*>(g.alloc(sizeof(float) * pix * wl.ldc, true));
                    wl.dcols = static_cast<float*>(g.alloc(sizeof(float) * pix * wl.ldk, true));
                }
            } else {
                wl.delta_img = wl.ldd;
            }
            wl.delta = static_cast<float*>(g.alloc(sizeof(float) * ring_rows_ * wl.delta_img, true));
            // bias-gradient partials: dense colsum chunks, or one row per (micro-batch, merge block) for conv
            // (proposed policy: per-micro-batch column sums, [m][colsum chunks of one micro-batch])
            wl.cc_mb = colsum_chunks(static_cast<long long>(mb_sizes_[0]) * (wl.delta_img / wl.ldd));
            const long long prow = std::max<long long>(
                li.kind == 1 ? std::max<long long>(static_cast<long long>(cfg_.m) * conv_merge_blocks() * li.Ho() * li.Wo(),
                                                   kColsumChunks)
                             : kColsumChunks,
                static_cast<long long>(cfg_.m) * wl.cc_mb);
            wl.partial = static_cast<float*>(g.alloc(sizeof(float) * prow * wl.u));
            // upload the shard rows [lo, hi) (train_partitioned.cpp:168-169), fp64 -> fp32;
            // conv rows [k][k][C_in] go to the GEMM layout [k*k][ck] (zero-padded channels)
            tmp.assign(static_cast<size_t>(wl.u) * wl.ldw, 0.f);
            const double* Wl = host_W_[wl.layer - 1];
            for (int r = 0; r < wl.u; ++r) {
                const double* src = Wl + static_cast<size_t>(wl.lo + r) * hc;
                float* dst = tmp.data() + static_cast<size_t>(r) * wl.ldw;
                if (li.kind == 1 && !li.im2col && !li.generic) {
                    for (int t = 0; t < li.ksz * li.ksz; ++t)
                        for (int c = 0; c < li.in_units; ++c)
                            dst[t * li.ck() + c] = static_cast<float>(src[t * li.in_units + c]);
                } else {
                    for (int c = 0; c < hc; ++c) dst[c] = static_cast<float>(src[c]);
                }
            }
            check(cudaSetDevice(w.gpu), "cudaSetDevice");
            check(cudaMemcpy(wl.W, tmp.data(), sizeof(float) * tmp.size(), cudaMemcpyHostToDevice), "upload W");
            if (li.dense_conv) {
                wl.dcg.ldw = wl.ldw;
                check(launch_dense_conv_expand(wl.dcg, wl.W, wl.Wx, nullptr), "expand Wx");
                check(cudaDeviceSynchronize(), "expand Wx");
            }
            std::vector<float> bb(wl.u);
            for (int r = 0; r < wl.u; ++r) bb[r] = static_cast<float>(host_b_[wl.layer - 1][wl.lo + r]);
            check(cudaMemcpy(wl.bias, bb.data(), sizeof(float) * wl.u, cudaMemcpyHostToDevice), "upload b");
            wl.delta_ready.assign(cfg_.m, {});
            wl.fwd_op.assign(cfg_.m, -1);
            wl.dgrad_op.assign(cfg_.m, -1);
        }
    }
    // contributor slots: multi-contributor dense merges, every conv merge
    for (int l = 2; l <= L; ++l) {
        int ncontrib = 0;
        for (int wi : layer_workers_[l]) ncontrib += workers_[wi]->at(l).contributor;
        const LayerInfo& dl = net_.info[l - 2];
        const LayerInfo& cl = net_.info[l - 1];
        if (dl.kind == 0 && ncontrib < 2) continue;
        for (int wi : layer_workers_[l - 1]) {
            Worker& w = *workers_[wi];
            WLayer& wl = w.at(l - 1);
            Gpu& g = gpu_of(w.gpu);
            long long rows = ring_rows_;
            if (dl.kind == 0) {
                wl.slot_ld = wl.ldd;
            } else if (cl.kind == 1) {  // conv consumer: pixel-major over the pooled grid
                wl.slot_ld = ld_of(wl.u);
                rows = ring_rows_ * dl.Hq() * dl.Wq();
            } else {  // dense consumer: CHW-flatten columns of this shard's channels
                wl.slot_ld = ld_of(wl.u * dl.Hq() * dl.Wq());
            }
            for (int k = 0; k < ncontrib; ++k)
                wl.slots.push_back(static_cast<float*>(g.alloc(sizeof(float) * rows * wl.slot_ld, true)));
        }
    }
    // NCCL merge backend buffers (dense layers whose merges go through NCCL)
    for (int l = 1; l < L; ++l) {
        if (!nccl_layer(l)) continue;
        const int gsz = static_cast<int>(layer_workers_[l].size());
        for (int wi : layer_workers_[l]) {
            Worker& w = *workers_[wi];
            Gpu& g = gpu_of(w.gpu);
            WLayer& wl = w.at(l);
            const size_t blk = static_cast<size_t>(ring_rows_) * wl.u;
            wl.ag_send = static_cast<float*>(g.alloc(sizeof(float) * blk, true));
            wl.ag_recv = static_cast<float*>(g.alloc(sizeof(float) * blk * gsz, true));
            wl.rs_recv = static_cast<float*>(g.alloc(sizeof(float) * blk, true));
            // the dgrad of layer l + 1 on this device packs its partial per destination rank
            WLayer& wn = w.at(l + 1);
            wn.rs_send = static_cast<float*>(g.alloc(sizeof(float) * blk * gsz, true));
        }
    }
    for (auto& gp : gpus_) {
        cudaSetDevice(gp->ordinal);
        check(cudaDeviceSynchronize(), "alloc");
    }
}

int Session::add_op(int gpu, cudaStream_t s, std::function<cudaError_t()> f, std::vector<int> deps,
                    int kernels, int kind, double flops) {
    // timing probes only (wrong results): PPB_PROBE_SKIP = bitmask of op kinds
    // whose launches are dropped from the step (dependencies are kept)
    const unsigned skip = dev_knob_uint("PPB_PROBE_SKIP");
    if (kind > 0 && (skip >> kind) & 1u) {
        f = nullptr;
        kernels = 0;
    }
    Op op;
    op.kind = kind;
    op.flops = flops;
    op.layer = cur_layer_;
    op.info = (kind == OP_FWD_GEMM || kind == OP_DGRAD_GEMM || kind == OP_WGRAD_GEMM) ? cur_info_ : 0;
    op.gpu = gpu;
    op.stream = s;
    op.launch = std::move(f);
    op.deps = std::move(deps);
    op.kernels = kernels;
    op.mb = cur_mb_;
    check(cudaSetDevice(gpu), "cudaSetDevice");
    check(cudaEventCreateWithFlags(&op.ev, cudaEventDisableTiming), "event");
    ops_.push_back(std::move(op));
    return static_cast<int>(ops_.size()) - 1;
}

void Session::build_ops() {
    const int L = net_.L();
    const int F = net_.dims[L];
    const bool softmax = net_.acts[L - 1] == 2;
    const int m = cfg_.m;
    const bool tf32 = cfg_.precision == 0;
    Gpu& g0 = *gpus_[0];
    begin_op_ = add_op(g0.ordinal, g0.main, nullptr, {}, 0);

    auto gemm_launch = [tf32](TcGemmPlan* p, GemmDesc* d, cudaStream_t s) -> std::function<cudaError_t()> {
        if (tf32) return [p, d, s]() { return tc_gemm_launch(*p, s); };
        return [d, s]() { return simt_gemm_launch(*d, s); };
    };
    // kernels per GEMM launch (the split-K reduction is a second kernel)
    auto nk = [tf32](const TcGemmPlan& p) { return tf32 && p.sk.splits > 1 && !p.sk.fixup ? 2 : 1; };
    auto prepare = [&](GemmDesc& d, TcGemmPlan& p, int gpu) {
        if (!tf32) return;
        char err[256];
        Gpu* g = &gpu_of(gpu);
        WsAlloc ws = [g](size_t n) { return static_cast<float*>(g->alloc(sizeof(float) * n)); };
        if (!tc_gemm_prepare(d, &p, 0, err, sizeof(err), ws)) throw std::runtime_error(std::string("GEMM setup: ") + err);
        cur_info_ = p.bn | (p.cg << 10) | (p.sk.splits << 12) | (p.halo << 24);
    };
    auto module_of_layer = [&](int l) -> const SubModule& {
        for (const SubModule& sm : plan_.subs)
            if (l >= sm.first_layer && l <= sm.last_layer) return sm;
        throw std::runtime_error("internal: no module for layer");
    };
    auto contributors = [&](int l) {
        std::vector<int> c;
        for (int wi : layer_workers_[l])
            if (workers_[wi]->at(l).contributor) c.push_back(wi);
        return c;
    };

    // pre-size the plan/desc vectors (pointers into them are captured)
    for (auto& wp : workers_)
        for (WLayer& wl : wp->layers) {
            wl.p_fwd.resize(m);
            wl.d_fwd.resize(m);
            wl.p_dgrad.resize(m);
            wl.d_dgrad.resize(m);
        }

    // per (layer, micro-batch): ops whose completion makes a_layer (or q) of
    // that micro-batch available on a given GPU
    std::vector<std::vector<std::map<int, std::vector<int>>>> act_ready(
        L + 1, std::vector<std::map<int, std::vector<int>>>(m));
    std::vector<std::vector<int>> loss_ops(m);

    // weight-gradient GEMM of one worker layer (dW = delta^T . a_{l-1}) over
    // micro-batch j, or over all b rows of the batch when j < 0 (the
    // stash_all executor: one GEMM per layer, K = every row); epilogue = the
    // update (SGD on W, or plain dWx for a dense-conv layer)
    auto wgrad_desc = [&](Worker& w, WLayer& wl, int j, GemmDesc& d, double* wfl, long long* bias_rows) {
        const int l = wl.layer;
        const int fi = net_.dims[l - 1];
        const LayerInfo& li = net_.info[l - 1];
        Gpu& g = gpu_of(w.gpu);
        const int rows = j < 0 ? cfg_.batch : mb_sizes_[j];
        const long long so = j < 0 ? 0 : soff(j);
        const float* delta = wl.delta + so * wl.delta_img;
        const float* ain = act_buf(w.gpu, l - 1) + (j < 0 ? 0 : aoff(l - 1, j)) * img_elems(l - 1);
        d = GemmDesc{};
        *bias_rows = rows;
        if (li.kind == 1) {
            ConvShape cs;
            cs.N = rows;
            cs.H = li.H;
            cs.W = li.W;
            cs.C = li.in_units;
            cs.ksz = li.ksz;
            cs.pad = li.pad;
            cs.u = wl.u;
            if (li.dense_conv) {  // dWx = delta^T . a over the images (K = images); folded by the update
                const int P = li.Ho() * li.Wo(), Q = li.H * li.W;
                d.a = Operand{delta, rows, P * wl.u, wl.delta_img, true};
                d.b = Operand{ain, rows, Q * li.in_units, img_elems(l - 1), true};
                d.M = P * wl.u;
                d.N = Q * li.in_units;
                d.K = rows;
            } else if (li.dense_delta) {  // dense wgrad: K = output pixels, unpadded error signal x im2col rows
                const int kc = li.ksz * li.ksz * li.in_units;
                const int pix = rows * li.Ho() * li.Wo();
                const float* colsp = li.generic ? wl.cols + so * li.Ho() * li.Wo() * wl.ldc : ain;
                const long long ldc = li.generic ? wl.ldc : lay_[l - 1].ld;
                d.a = Operand{delta, pix, wl.u, wl.ldd, true};
                d.b = Operand{colsp, pix, kc, ldc, true};
                d.M = wl.u;
                d.N = kc;
                d.K = pix;
                if (wl.u < 128 && kc > wl.u) {  // dW^T: the wide side fills the 128-row tiles
                    std::swap(d.a, d.b);
                    std::swap(d.M, d.N);
                }
            } else if (li.im2col) {  // B = im2col rows (pixel-major, MN = k*k*C)
                d = conv_wgrad_desc(cs, delta, wl.ldd, ain, lay_[l - 1].ld, false);
                const int kc = li.ksz * li.ksz * li.in_units;
                d.b = Operand{ain, rows * li.Ho() * li.Wo(), kc, lay_[l - 1].ld, true};
                d.N = kc;
            } else {
                d = conv_wgrad_desc(cs, delta, wl.ldd, ain, lay_[l - 1].ld, wl.u < 128);
            }
            *wfl = li.dense_conv ? 2.0 * rows * li.Ho() * li.Wo() * wl.u * li.H * li.W * li.in_units  // executed
                                 : 2.0 * rows * li.Ho() * li.Wo() * wl.u * li.ksz * li.ksz * li.in_units;
            *bias_rows = static_cast<long long>(rows) * (wl.delta_img / wl.ldd);  // zero borders add nothing
        } else {
            d.a = Operand{delta, rows, wl.u, wl.ldd, true};
            d.b = Operand{ain, rows, fi, lay_[l - 1].ld, true};
            d.M = wl.u;
            d.N = fi;
            d.K = rows;
            if (wl.u < 128 && fi > wl.u) {  // dW^T: the wide side fills the 128-row tiles
                std::swap(d.a, d.b);
                std::swap(d.M, d.N);
            }
            *wfl = 2.0 * wl.u * fi * static_cast<double>(rows);
        }
        const bool wt = d.M != wl.u;
        d.epi = EpiParams{};
        d.epi.mode = EPI_SGD;
        d.epi.W = wl.W;
        d.epi.ldw = wl.ldw;
        d.epi.sgd_t = wt ? 1 : 0;
        d.epi.alpha = &g.st->alpha;
        d.epi.inv_b = 1.f / static_cast<float>(cfg_.batch);
        d.epi.flag = &g.st->diverge_flag;
        if (li.dense_conv) {  // plain dWx; the fold kernel applies SGD to W and re-expands Wx
            d.epi = EpiParams{};
            d.epi.mode = EPI_STORE;
            d.epi.dst[d.epi.ndst++] = wl.dWx;
            d.epi.ldd = wl.ldwx;
        }
    };
    // conv layers whose bias-gradient partials come with the backward merges
    // ([j][merge block][u] rows written by conv_merge / the EPI_MERGE epilogue)
    auto bias_from_merge = [&](const WLayer& wl) { return net_.info[wl.layer - 1].kind == 1 && !wl.db_colsum; };
    // proposed memory policy: micro-batch j's weight gradients as soon as its
    // backward has produced every error signal (raw partial sums into the
    // layer's slices for micro-batch j, no update), and its bias column sums
    std::vector<int> bjoin(m, -1);
    auto per_mb_wgrads = [&](int j, int first_op) {
        for (auto& wp : workers_) {
            Worker& w = *wp;
            for (auto wit = w.layers.rbegin(); wit != w.layers.rend(); ++wit) {
                WLayer& wl = *wit;
                cur_layer_ = wl.layer;
                if (wl.p_wg.empty()) {
                    wl.p_wg.resize(m);
                    wl.d_wg.resize(m);
                    wl.wg_op.clear();
                }
                GemmDesc& d = wl.d_wg[j];
                double wfl;
                long long brows;
                wgrad_desc(w, wl, j, d, &wfl, &brows);
                d.partial_out = 1;
                d.force_splits = j == 0 ? 0 : wl.acc_slices;
                Gpu* g = &gpu_of(w.gpu);
                WLayer* wlp = &wl;
                const int mm = m;
                WsAlloc ws = [g, wlp, j, mm](size_t n) -> float* {
                    if (j == 0) {
                        wlp->acc_ws = static_cast<float*>(g->alloc(sizeof(float) * n * mm));
                        return wlp->acc_ws;
                    }
                    return wlp->acc_ws + static_cast<long long>(j) * wlp->acc_slices * wlp->p_wg[0].sk.stride;
                };
                char err[256];
                if (!tc_gemm_prepare(d, &wl.p_wg[j], 0, err, sizeof(err), ws))
                    throw std::runtime_error(std::string("GEMM setup: ") + err);
                cur_info_ = wl.p_wg[j].bn | (wl.p_wg[j].cg << 10) | (wl.p_wg[j].sk.splits << 12);
                if (j == 0) wl.acc_slices = wl.p_wg[0].sk.splits;
                const int gop = add_op(w.gpu, w.su, gemm_launch(&wl.p_wg[j], &wl.d_wg[j], w.su), wl.delta_ready[j], 1,
                                       OP_WGRAD_GEMM, wfl);
                wl.wg_op.push_back(gop);
                if (!bias_from_merge(wl)) {
                    const float* dj = wl.delta + soff(j) * wl.delta_img;
                    const long long ldd = wl.ldd;
                    const int u = wl.u;
                    float* part = wl.partial + static_cast<long long>(j) * wl.cc_mb * wl.u;
                    cudaStream_t s = w.su;
                    wl.wg_op.push_back(add_op(w.gpu, s, [=]() { return launch_colsum(dj, ldd, brows, u, part, s); },
                                              wl.delta_ready[j], 1, OP_BIAS));
                }
            }
        }
        std::vector<int> all;
        for (int i = first_op; i < static_cast<int>(ops_.size()); ++i) all.push_back(i);
        bjoin[j] = add_op(g0.ordinal, g0.main, nullptr, all, 0);
    };

    // ---------------- forward of micro-batch j (train_partitioned.cpp:245-419)
    auto forward = [&](int j) {
        cur_mb_ = j;
        const int rows = mb_sizes_[j];
        const long long off = mb_off_[j];  // batch rows (X, labels, per-sample loss)
        const long long so = soff(j);      // stash slot rows (activations l >= 1, error signals, ...)
        for (int l = 1; l <= L; ++l) {
            cur_layer_ = l;
            const SubModule& sm = module_of_layer(l);
            const bool last_in_module = l == sm.last_layer;
            const bool boundary_concat = last_in_module && sm.index < plan_.Z() &&
                                         plan_.boundaries[sm.index - 1] == kConcat;
            const SubModule* next = sm.index < plan_.Z() ? &plan_.subs[sm.index] : nullptr;
            std::set<int> dest_gpus;
            for (int wi : layer_workers_[l]) dest_gpus.insert(workers_[wi]->gpu);
            int hub_gpu = -1;
            if (l < L) {
                if (boundary_concat) {
                    hub_gpu = device_map_[next->devices.front() - 1];
                    dest_gpus.insert(hub_gpu);
                } else {
                    for (int wi : layer_workers_[l + 1]) dest_gpus.insert(workers_[wi]->gpu);
                }
            }
            std::vector<int> produced;
            const LayerInfo& li = net_.info[l - 1];
            for (int wi : contributors(l)) {
                Worker& w = *workers_[wi];
                WLayer& wl = w.at(l);
                const int fi = net_.dims[l - 1];
                GemmDesc& d = wl.d_fwd[j];
                std::vector<int> deps;
                if (l == 1) {
                    deps.push_back(begin_op_);
                } else {
                    auto it = act_ready[l - 1][j].find(w.gpu);
                    if (it != act_ready[l - 1][j].end()) deps.insert(deps.end(), it->second.begin(), it->second.end());
                }
                if (l == w.layers.front().layer && cfg_.gate > 0 && j - cfg_.gate >= 0 &&
                    w.last_bwd[j - cfg_.gate] >= 0)
                    deps.push_back(w.last_bwd[j - cfg_.gate]);  // schedule.cpp:293-296
                // proposed policy: micro-batch j takes the stash slots of j - ring,
                // free once that micro-batch's whole backward (wgrads included) ran
                if (l == w.layers.front().layer && ring_ < m && j - ring_ >= 0) deps.push_back(bjoin[j - ring_]);
                if (li.kind == 1) {
                    // implicit-GEMM conv over the padded NHWC input of this micro-batch
                    ConvShape cs;
                    cs.N = rows;
                    cs.H = li.H;
                    cs.W = li.W;
                    cs.C = li.in_units;
                    cs.ksz = li.ksz;
                    cs.pad = li.pad;
                    cs.u = wl.u;
                    if (li.dense_conv) {  // dense layer over all positions with the expanded weight
                        const int P = li.Ho() * li.Wo(), Q = li.H * li.W;
                        d = GemmDesc{};
                        d.a = Operand{act_buf(w.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1), rows, Q * li.in_units,
                                      img_elems(l - 1), false};
                        d.b = Operand{wl.Wx, P * wl.u, Q * li.in_units, wl.ldwx, false};
                        d.M = rows;
                        d.N = P * wl.u;
                        d.K = Q * li.in_units;
                    } else if (li.generic) {  // per-step im2col rows of the padded input, then a dense GEMM
                        const ActLayout& a = lay_[l - 1];
                        const float* x = act_buf(w.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1);
                        float* cols = wl.cols + so * li.Ho() * li.Wo() * wl.ldc;
                        const int hp = a.hp, wp = a.wp, C = li.in_units, k = li.ksz, Ho = li.Ho(), Wo = li.Wo(),
                                  st1 = li.stride;
                        const long long ldx = a.ld, ldc = wl.ldc;
                        cudaStream_t st = w.sf;
                        const int iop = add_op(w.gpu, st, [=]() {
                            return launch_im2col_act(x, rows, hp, wp, ldx, C, k, Ho, Wo, cols, ldc, st, st1);
                        }, deps, 1, OP_POOL);
                        deps = {iop};
                        const int kc = k * k * C;
                        d = GemmDesc{};
                        d.a = Operand{cols, rows * Ho * Wo, kc, ldc, false};
                        d.b = Operand{wl.W, wl.u, kc, wl.ldw, false};
                        d.M = rows * Ho * Wo;
                        d.N = wl.u;
                        d.K = kc;
                    } else if (li.im2col) {  // dense GEMM over the im2col rows
                        const int kc = li.ksz * li.ksz * li.in_units;
                        const int prow = rows * li.Ho() * li.Wo();
                        d = GemmDesc{};
                        d.a = Operand{act_buf(w.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1), prow, kc, lay_[l - 1].ld, false};
                        d.b = Operand{wl.W, wl.u, kc, wl.ldw, false};
                        d.M = prow;
                        d.N = wl.u;
                        d.K = kc;
                    } else {
                        d = conv_fwd_desc(cs, act_buf(w.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1), lay_[l - 1].ld, wl.W);
                    }
                    d.epi = EpiParams{};
                    d.epi.mode = EPI_STORE;
                    d.epi.bias = wl.bias;
                    d.epi.relu = li.act == 1 && !li.special();  // residual / avg: the activation follows the shortcut
                    const long long pix = static_cast<long long>(li.Ho()) * li.Wo();
                    // residual layer without pooling: the shortcut add (identity or option A) and
                    // the ReLU run in the GEMM epilogue, which stores straight into the
                    // consumers (no U round trip, no residual_act pass); the backward mask
                    // then reads the activation (relu(u) > 0 <=> u > 0)
                    static const bool no_res_fuse = dev_knob("PPB_NO_RES_FUSE");  // A/B switch
                    bool res_fuse = false;
                    if (!no_res_fuse && li.res_from > 0 && !li.pool_avg && li.pool == 1 && li.act == 1 &&
                        !li.dense_conv && lay_[l].kind == 0) {
                        const int sl = li.res_from;
                        const LayerInfo& ls = net_.info[sl - 1];
                        // identity (f = 1, C_s = C_l) or option A (f = 2, C_s <= C_l)
                        const int f = ls.Hq() / li.Ho();
                        res_fuse = f >= 1 && ls.Hq() == f * li.Ho() && ls.Wq() == f * li.Wo() &&
                                   ls.out_units <= li.out_units && lay_[sl].kind == 0;
                    }
                    if (res_fuse) {
                        const int sl = li.res_from;
                        const ActLayout& sa = lay_[sl];
                        d.epi.relu = 1;
                        d.epi.rs_src = act_buf(w.gpu, sl) + so * img_elems(sl);
                        d.epi.rs_ld = sa.ld;
                        d.epi.rs_hp = sa.hp;
                        d.epi.rs_wp = sa.wp;
                        d.epi.rs_pad = sa.pad;
                        d.epi.rs_col0 = wl.lo;
                        d.epi.rs_f = net_.info[sl - 1].Hq() / li.Ho();
                        d.epi.rs_C = net_.info[sl - 1].out_units;
                        d.force_splits = 1;  // the split-K reduction kernel has no shortcut term
                        auto it = act_ready[sl][j].find(w.gpu);
                        if (it != act_ready[sl][j].end()) deps.insert(deps.end(), it->second.begin(), it->second.end());
                        wl.u_written = false;
                    }
                    if (wl.U != nullptr && !res_fuse) {  // pre-pool output, then pool / relayout
                        d.epi.dst[d.epi.ndst++] = wl.U + so * pix * wl.ldu;
                        d.epi.ldd = wl.ldu;
                    } else {  // straight into every consumer GPU's padded NHWC input
                        const ActLayout& a = lay_[l];
                        d.epi.remap = 1;
                        d.epi.r_wo = li.Wo();
                        d.epi.r_howo = static_cast<int>(pix);
                        d.epi.r_hp = a.hp;
                        d.epi.r_wp = a.wp;
                        d.epi.r_pad = a.pad;
                        d.epi.ldd = a.ld;
                        d.epi.col0 = wl.lo;
                        for (int ord : dest_gpus) d.epi.dst[d.epi.ndst++] = act_buf(ord, l) + so * img_elems(l);
                    }
                    if (li.dense_conv) {  // segmented columns (p, c): unpadded per-pixel rows of the destination
                        d.epi.remap = 0;
                        d.epi.seg_w = wl.u;
                        if (wl.U != nullptr) {
                            d.epi.seg_pitch = wl.ldu;
                            d.epi.ldd = pix * wl.ldu;
                            d.epi.col0 = 0;
                        } else {
                            d.epi.seg_pitch = lay_[l].ld;
                            d.epi.ldd = img_elems(l);
                            d.epi.col0 = wl.lo;
                        }
                    }
                    // 2x2 max-pool fused into the epilogue when each warp's 32 rows hold
                    // whole windows (grid width <= 16); the GEMM must end up unsplit and
                    // on the tc kernel, else the pool kernel runs as before
                    static const bool no_pool_fuse = dev_knob("PPB_NO_POOL_FUSE");
                    // Grid width 32 (VGG conv2 / conv4 on the rank-4 path): 128-row tiles are
                    // 4 image rows, the windows span warp pairs (pl_on 3, TMA-store staging)
                    const int Wo1 = li.Wo(), Ho1 = li.Ho();
                    const bool in_warp = Wo1 >= 2 && 32 % (2 * Wo1) == 0 && (pix % 32 == 0 || 32 % pix == 0);
                    static const bool no_pool_pair = dev_knob("PPB_NO_POOL_PAIR");  // A/B switch
                    const bool pair = !no_pool_pair && Wo1 == 32 && pix % 128 == 0 && lay_[l].kind != 1 && wl.u >= 32;
                    if (tf32 && !no_pool_fuse && li.pool == 2 && wl.U != nullptr && !li.dense_conv && wl.argmax &&
                        Ho1 % 2 == 0 && (in_warp || pair)) {
                        const ActLayout& a = lay_[l];
                        const bool pool_smem = dev_knob("PPB_POOL_SMEM");
                        d.epi.pl_on = !in_warp ? 3 : pool_smem ? 2 : 1;
                        d.epi.pl_wo = Wo1;
                        d.epi.pl_ho = Ho1;
                        for (int ord : dest_gpus) d.epi.pl_dst[d.epi.pl_ndst++] = act_buf(ord, l) + so * img_elems(l);
                        d.epi.pl_kind = a.kind == 1 ? 1 : 0;
                        d.epi.pl_ld = a.ld;
                        d.epi.pl_hp = a.hp;
                        d.epi.pl_wp = a.wp;
                        d.epi.pl_pad = a.pad;
                        d.epi.pl_col0 = wl.lo;
                        d.epi.pl_arg = wl.argmax + so * li.Hq() * li.Wq() * wl.u;
                        d.epi.pl_uch = wl.u;
                    }
                    prepare(d, wl.p_fwd[j], w.gpu);
                    bool pool_fused = false;
                    if (d.epi.pl_on) {
                        pool_fused = wl.p_fwd[j].halo == 0 && wl.p_fwd[j].sk.splits == 1 &&
                                     (d.epi.pl_on != 3 || wl.p_fwd[j].ts.n > 0);
                        if (!pool_fused) wl.p_fwd[j].epi.pl_on = 0;
                        if (pool_fused && d.epi.pl_on == 3) wl.u_written = false;  // pre-pool rows never stored
                    }
                    const double fl = li.dense_conv ? 2.0 * rows * pix * wl.u * li.H * li.W * li.in_units  // executed
                                                    : 2.0 * rows * pix * wl.u * li.ksz * li.ksz * li.in_units;
                    int op = add_op(w.gpu, w.sf, gemm_launch(&wl.p_fwd[j], &wl.d_fwd[j], w.sf), deps, nk(wl.p_fwd[j]), OP_FWD_GEMM, fl);
                    if (wl.U != nullptr && !pool_fused && li.special() && !res_fuse) {
                        // residual extension: U + shortcut -> act -> (average pool) -> consumers
                        ActLayout out = lay_[l];
                        out.col0 = wl.lo;
                        PoolDsts pd;
                        for (int ord : dest_gpus) pd.ptr[pd.n++] = act_buf(ord, l) + so * img_elems(l);
                        SkipSrc sk;
                        std::vector<int> rdeps{op};
                        if (li.res_from > 0) {
                            const int sl = li.res_from;
                            sk.a = act_buf(w.gpu, sl) + so * img_elems(sl);
                            sk.lay = lay_[sl];
                            sk.f = net_.info[sl - 1].Hq() / li.Ho();
                            sk.C = net_.info[sl - 1].out_units;
                            auto it = act_ready[sl][j].find(w.gpu);
                            if (it != act_ready[sl][j].end()) rdeps.insert(rdeps.end(), it->second.begin(), it->second.end());
                        }
                        float* U = wl.U + so * pix * wl.ldu;
                        const long long ldu = wl.ldu;
                        const int Ho = li.Ho(), Wo = li.Wo(), u = wl.u, c0 = wl.lo, pool = li.pool, relu = li.act == 1;
                        // launch_residual_act keeps U + shortcut only for pooled outputs: the
                        // backward mask of the others reads the activation (mask_kind 2)
                        if (relu && pool == 1) wl.u_written = false;
                        cudaStream_t st = w.sf;
                        op = add_op(w.gpu, st, [=]() {
                            return launch_residual_act(U, ldu, rows, Ho, Wo, u, c0, relu, pool, sk, out, pd, st);
                        }, rdeps, 1, OP_POOL);
                    } else if (wl.U != nullptr && !pool_fused && !res_fuse) {
                        ActLayout out = lay_[l];
                        out.col0 = wl.lo;
                        PoolDsts pd;
                        for (int ord : dest_gpus) pd.ptr[pd.n++] = act_buf(ord, l) + so * img_elems(l);
                        const float* U = wl.U + so * pix * wl.ldu;
                        const long long ldu = wl.ldu;
                        unsigned char* am = wl.argmax ? wl.argmax + so * li.Hq() * li.Wq() * wl.u : nullptr;
                        const int Ho = li.Ho(), Wo = li.Wo(), u = wl.u, pool = li.pool;
                        cudaStream_t st = w.sf;
                        op = add_op(w.gpu, st, [=]() {
                            return launch_pool_fwd(U, ldu, rows, Ho, Wo, u, pool, am, out, pd, st);
                        }, {op}, 1, OP_POOL);
                    }
                    wl.fwd_op[j] = op;
                    produced.push_back(op);
                    continue;
                }
                d.a = Operand{act_buf(w.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1), rows, fi, lay_[l - 1].ld, false};
                d.b = Operand{wl.W, wl.u, fi, wl.ldw, false};
                d.M = rows;
                d.N = wl.u;
                d.K = fi;
                d.epi = EpiParams{};
                d.epi.mode = EPI_STORE;
                d.epi.bias = wl.bias;
                d.epi.relu = net_.acts[l - 1] == 1;
                d.epi.col0 = wl.lo;
                d.epi.ldd = ld_of(net_.dims[l]);
                if (nccl_layer(l)) {  // NCCL backend: the shard output stays local, packed [rows][u]
                    d.epi.col0 = 0;
                    d.epi.ldd = wl.u;
                    d.epi.dst[d.epi.ndst++] = wl.ag_send + so * wl.u;
                } else {
                    for (int ord : dest_gpus) {
                        float* base = (l == L && softmax) ? q_buf(ord) : act_buf(ord, l);
                        d.epi.dst[d.epi.ndst++] = base + so * d.epi.ldd;
                    }
                }
                prepare(d, wl.p_fwd[j], w.gpu);
                const int op = add_op(w.gpu, w.sf, gemm_launch(&wl.p_fwd[j], &wl.d_fwd[j], w.sf), deps, nk(wl.p_fwd[j]),
                                      OP_FWD_GEMM, 2.0 * rows * wl.u * fi);
                wl.fwd_op[j] = op;
                produced.push_back(op);
            }
            for (int ord : dest_gpus) act_ready[l][j][ord] = produced;
            if (nccl_layer(l)) {
                // ncclAllGather of the packed shard outputs (one group over the
                // sub-module's ranks, each on its worker's forward stream, after
                // its GEMM), then each GPU lays the [g][rows][u] result out as the
                // activation rows the next layer reads
                const auto& ws = layer_workers_[l];
                const int gsz = static_cast<int>(ws.size());
                std::vector<const float*> snd;
                std::vector<float*> rcv;
                std::vector<cudaStream_t> sts;
                for (int wi : ws) {
                    WLayer& wl = workers_[wi]->at(l);
                    snd.push_back(wl.ag_send + so * wl.u);
                    rcv.push_back(wl.ag_recv + so * gsz * wl.u);
                    sts.push_back(workers_[wi]->sf);
                }
                const NcclGroup* grp = nccl_[module_index(l) - 1].get();
                const int u = workers_[ws.front()]->at(l).u;
                const size_t count = static_cast<size_t>(rows) * u;
                Worker& w0 = *workers_[ws.front()];
                const int cop = add_op(w0.gpu, w0.sf, [=]() { return nccl_all_gather(*grp, snd, rcv, count, sts); },
                                       produced, 0, OP_COPY);
                const long long ld = ld_of(net_.dims[l]);
                for (size_t k = 0; k < ws.size(); ++k) {
                    Worker& w = *workers_[ws[k]];
                    const float* rv = rcv[k];
                    float* dst = act_buf(w.gpu, l) + so * ld;
                    cudaStream_t st = w.sf;
                    act_ready[l][j][w.gpu] = {add_op(w.gpu, st, [=]() {
                        return launch_unpack_gather(rv, gsz, rows, u, dst, ld, st);
                    }, {cop}, 1, OP_COPY)};
                }
            }
            if (l < L && boundary_concat) {
                // concat_repartition: gather at the hub, then broadcast the full
                // activation to the other consumer GPUs (:258-271, :357-362)
                std::set<int> consumers;
                for (int wi : layer_workers_[l + 1]) consumers.insert(workers_[wi]->gpu);
                Gpu& hub = gpu_of(hub_gpu);
                const long long ld = img_elems(l);
                for (int ord : consumers) {
                    if (ord == hub_gpu) continue;
                    float* src = act_buf(hub_gpu, l) + so * ld;
                    float* dst = act_buf(ord, l) + so * ld;
                    const size_t bytes = sizeof(float) * rows * ld;
                    const int src_dev = hub_gpu, dst_dev = ord;
                    cudaStream_t s = hub.main;
                    const int op = add_op(hub_gpu, s, [=]() { return cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes, s); },
                                          produced, 0, OP_COPY);
                    act_ready[l][j][ord] = {op};
                }
            }
        }
        // loss head on every GPU holding last-module workers
        std::set<int> head_gpus;
        for (int wi : layer_workers_[L]) head_gpus.insert(workers_[wi]->gpu);
        for (int ord : head_gpus) {
            Gpu& g = gpu_of(ord);
            LossTargets t;
            for (int wi : layer_workers_[L]) {
                Worker& w = *workers_[wi];
                if (w.gpu != ord) continue;
                WLayer& wl = w.at(L);
                t.lo[t.n] = wl.lo;
                t.hi[t.n] = wl.hi;
                t.delta[t.n] = wl.delta + so * wl.ldd;
                t.ld[t.n] = wl.ldd;
                ++t.n;
            }
            const float* in = (softmax ? g.q : act_buf(ord, L)) + so * ld_of(F);
            const long long ldin = ld_of(F);
            const bool write = ord == main_gpu_;
            double* lr = write ? g.loss_row + off : nullptr;
            int* cr = write ? g.correct_row + off : nullptr;
            const int* lab = g.labels + off;
            const int kind = cfg_.loss;
            const int relu_last = net_.acts[L - 1] == 1;
            cudaStream_t s = g.main;
            const int op = add_op(ord, s, [=]() {
                return launch_loss_head(in, ldin, rows, F, lab, kind, relu_last, t, lr, cr, s);
            }, act_ready[L][j][ord], 1, OP_LOSS);
            loss_ops[j].push_back(op);
            for (int wi : layer_workers_[L]) {
                Worker& w = *workers_[wi];
                if (w.gpu == ord) w.at(L).delta_ready[j] = {op};
            }
        }
    };

    // ---------------- backward of micro-batch j (train_partitioned.cpp:422-630)
    auto backward = [&](int j) {
        cur_mb_ = j;
        const int rows = mb_sizes_[j];
        const long long so = soff(j);  // stash slot rows of micro-batch j
        const int first_op = static_cast<int>(ops_.size());
        for (int l = L; l >= 2; --l) {
            cur_layer_ = l;
            const std::vector<int> contrib = contributors(l);
            const std::vector<int>& dests = layer_workers_[l - 1];
            const int fi = net_.dims[l - 1];
            const bool relu_below = net_.acts[l - 2] == 1;
            const bool single = contrib.size() == 1;
            std::vector<int> dgrad_ops;
            const LayerInfo& li = net_.info[l - 1];
            const LayerInfo& lb = net_.info[l - 2];
            if (lb.kind == 1) {
                // destination is a conv layer: every contributor scatters its
                // partial input gradient (conv: pixel-major over the pooled grid,
                // dense: CHW-flatten columns) into per-destination slots; the
                // destination sums them, routes through the pool argmax and
                // masks by its ReLU into its padded error signal.
                const int hw = lb.Hq() * lb.Wq();
                const bool res_dest = lb.special() || skip_source(l - 1);  // residual-extension merge kernel
                // a residual / skip-source destination merges in the dgrad epilogue too when
                // it needs no average-pool routing and its shortcut gradient is an identity
                // (EPI_MERGE + mg_sg); its ReLU mask then comes from its activation, which
                // holds for residual layers (their U is not kept, relu(u) > 0 <=> u > 0)
                static const bool no_sg_fuse = dev_knob("PPB_NO_SG_FUSE");  // A/B switch
                WLayer* sg_src = nullptr;
                bool res_fusable = false;
                if (res_dest && !no_sg_fuse && !lb.pool_avg && lb.pool == 1 && contrib.size() == 1 &&
                    dests.size() == 1 && (!lb.special() || !workers_[dests[0]]->at(l - 1).u_written)) {
                    res_fusable = true;
                    if (const int r = res_consumer(l - 1)) {
                        const LayerInfo& lr = net_.info[r - 1];
                        const WLayer& dl0 = workers_[dests[0]]->at(l - 1);
                        for (int wi : layer_workers_[r]) {
                            WLayer& cand = workers_[wi]->at(r);
                            if (cand.contributor && cand.lo <= dl0.lo && dl0.hi <= cand.hi) sg_src = &cand;
                        }
                        res_fusable = sg_src != nullptr && lb.Hq() == lr.Ho() && lb.Wq() == lr.Wo() &&
                                      workers_[dests[0]]->gpu == workers_[contrib[0]]->gpu;
                    }
                }
                if (li.kind == 1 && !li.generic && !li.dense_conv && contrib.size() == 1 && dests.size() == 1 &&
                    fuse_merge_ && (!res_dest || res_fusable)) {
                    // one contributor, one destination: the merge (pool routing,
                    // ReLU mask, padded store) runs in the dgrad epilogue
                    Worker& w = *workers_[contrib[0]];
                    WLayer& wl = w.at(l);
                    Worker& dw = *workers_[dests[0]];
                    WLayer& dl = dw.at(l - 1);
                    GemmDesc& d = wl.d_dgrad[j];
                    ConvShape cs;
                    cs.N = rows;
                    cs.H = li.H;
                    cs.W = li.W;
                    cs.C = li.in_units;
                    cs.ksz = li.ksz;
                    cs.pad = li.pad;
                    cs.u = wl.u;
                    d = conv_dgrad_desc(cs, wl.delta + so * wl.delta_img, wl.ldd, wl.W);
                    d.epi = EpiParams{};
                    d.epi.mode = EPI_MERGE;
                    d.epi.mg_pool = lb.pool;
                    d.epi.mg_hg = lb.Hq();
                    d.epi.mg_wg = lb.Wq();
                    d.epi.mg_argmax = dl.argmax ? dl.argmax + so * hw * dl.u : nullptr;
                    d.epi.mg_uch = dl.u;
                    if (relu_below) {  // mask at the pooled pixel of the layer's output (consumer layout)
                        const ActLayout& a = lay_[l - 1];
                        d.epi.mg_mask = act_buf(dw.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1);
                        d.epi.mg_mld = a.ld;
                        d.epi.mg_mhp = a.hp;
                        d.epi.mg_mwp = a.wp;
                        d.epi.mg_mpad = a.pad;
                        d.epi.mg_mcol0 = dl.lo;
                    }
                    const int q = lb.dq();
                    d.epi.mg_d = dl.delta + so * dl.delta_img;
                    d.epi.mg_dld = dl.ldd;
                    d.epi.mg_dhp = lb.Ho() + 2 * q;
                    d.epi.mg_dwp = lb.Wo() + 2 * q;
                    d.epi.mg_dpad = q;
                    // bias-gradient partials of the layer below, same [j][merge block][u]
                    // layout the unfused conv_merge writes
                    d.epi.db_partial = dl.partial + static_cast<long long>(j) * conv_merge_blocks() * dl.u;
                    std::vector<int> gdeps = wl.delta_ready[j];
                    if (sg_src != nullptr) {  // the consuming residual layer's error signal (identity shortcut)
                        const LayerInfo& lr = net_.info[res_consumer(l - 1) - 1];
                        d.epi.mg_sg = sg_src->delta + so * sg_src->delta_img;
                        d.epi.mg_sld = sg_src->ldd;
                        d.epi.mg_spad = lr.dq();
                        d.epi.mg_shp = lr.Ho() + 2 * lr.dq();
                        d.epi.mg_swp = lr.Wo() + 2 * lr.dq();
                        d.epi.mg_sc0 = dl.lo - sg_src->lo;
                        gdeps.insert(gdeps.end(), sg_src->delta_ready[j].begin(), sg_src->delta_ready[j].end());
                    }
                    prepare(d, wl.p_dgrad[j], w.gpu);
                    if (!tf32 || wl.p_dgrad[j].epi.db_partial == nullptr) dl.db_colsum = true;
                    const double fl = 2.0 * rows * li.H * li.W * li.in_units * li.ksz * li.ksz * wl.u;
                    const int op = add_op(w.gpu, w.sb, gemm_launch(&wl.p_dgrad[j], &wl.d_dgrad[j], w.sb),
                                          gdeps, nk(wl.p_dgrad[j]), OP_DGRAD_GEMM, fl);
                    wl.dgrad_op[j] = op;
                    w.last_bwd[j] = std::max(w.last_bwd[j], op);
                    dl.merge_fused = true;
                    dl.delta_ready[j] = {op};
                    dw.last_bwd[j] = std::max(dw.last_bwd[j], op);
                    continue;
                }
                bool fused_dc = false;  // dense-conv dgrad performed the whole merge
                // 3x3 stride-2 generic conv, one contributor and one residual-extension
                // destination: the merge reads the column-space partial itself
                // (launch_conv_merge_res_col2im), no col2im pass and no slot round trip
                static const bool no_c2m_fuse = dev_knob("PPB_NO_COL2IM_MERGE");  // A/B switch
                const bool c2m = !no_c2m_fuse && li.kind == 1 && li.generic && !li.dense_conv && li.ksz == 3 &&
                                 li.stride == 2 && res_dest && lb.pool == 1 && !lb.pool_avg && contrib.size() == 1 &&
                                 dests.size() == 1 && workers_[dests[0]]->gpu == workers_[contrib[0]]->gpu;
                Col2imSrc c2m_src;
                for (size_t k = 0; k < contrib.size(); ++k) {
                    Worker& w = *workers_[contrib[k]];
                    WLayer& wl = w.at(l);
                    GemmDesc& d = wl.d_dgrad[j];
                    double fl;
                    long long rows_per_img;
                    if (li.kind == 1 && (li.generic || li.dense_conv)) {
                        // generic: dcols = delta . W (column space), then col2im into each
                        // destination's slot (its channel slice).  Dense conv: the
                        // input-gradient rows [img][(q, c)] = delta . Wx, then a k = 1
                        // col2im (channel-slice copy) into the slots.
                        const int kc = li.ksz * li.ksz * li.in_units;
                        const long long pix = static_cast<long long>(li.Ho()) * li.Wo();
                        const int Q = li.H * li.W;
                        d = GemmDesc{};
                        if (li.dense_conv) {
                            d.a = Operand{wl.delta + so * wl.delta_img, rows, static_cast<int>(pix) * wl.u, wl.delta_img,
                                          false};
                            d.b = Operand{wl.Wx, static_cast<int>(pix) * wl.u, Q * li.in_units, wl.ldwx, true};
                            d.M = rows;
                            d.N = Q * li.in_units;
                            d.K = static_cast<int>(pix) * wl.u;
                        } else {
                            d.a = Operand{wl.delta + so * wl.delta_img, static_cast<int>(rows * pix), wl.u, wl.ldd, false};
                            d.b = Operand{wl.W, wl.u, kc, wl.ldw, true};
                            d.M = static_cast<int>(rows * pix);
                            d.N = kc;
                            d.K = wl.u;
                        }
                        d.epi = EpiParams{};
                        d.epi.mode = EPI_STORE;
                        const long long drows = li.dense_conv ? 1 : pix;  // dcols rows per image
                        // dense conv, one destination owning every input channel with
                        // slot pitch C: the gradient rows [img][(q, c)] ARE its slot
                        WLayer& d0 = workers_[dests[0]]->at(l - 1);
                        const bool direct = li.dense_conv && dests.size() == 1 && d0.u == li.in_units &&
                                            d0.slot_ld == li.in_units;
                        // dense conv over an unpooled dense-layout layer below, one
                        // contributor: the whole merge (ReLU mask + bias partials, one
                        // partial row per (CTA, warp, position)) runs in the epilogue
                        const bool fused = direct && contrib.size() == 1 && fuse_merge_ && lb.pool == 1 &&
                                           lb.dq() == 0 && d0.ldd == li.in_units && tf32 && !res_dest;
                        if (fused) {
                            Worker& dw = *workers_[dests[0]];
                            d.epi.mode = relu_below ? EPI_MASK : EPI_STORE;
                            d.epi.dst[d.epi.ndst++] = d0.delta + so * d0.delta_img;
                            d.epi.ldd = d0.delta_img;
                            if (relu_below) {
                                d.epi.mask = act_buf(dw.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1);
                                d.epi.ldm = img_elems(l - 1);
                            }
                            d.epi.db_partial = d0.partial + static_cast<long long>(j) * conv_merge_blocks() * Q * d0.u;
                            prepare(d, wl.p_dgrad[j], w.gpu);
                            if (wl.p_dgrad[j].epi.db_partial == nullptr) d0.db_colsum = true;
                            d0.db_q = Q;
                            const double fl2 = 2.0 * rows * pix * wl.u * Q * li.in_units;
                            const int op = add_op(w.gpu, w.sb, gemm_launch(&wl.p_dgrad[j], &wl.d_dgrad[j], w.sb),
                                                  wl.delta_ready[j], nk(wl.p_dgrad[j]), OP_DGRAD_GEMM, fl2);
                            wl.dgrad_op[j] = op;
                            w.last_bwd[j] = std::max(w.last_bwd[j], op);
                            d0.merge_fused = true;
                            d0.delta_ready[j] = {op};
                            dw.last_bwd[j] = std::max(dw.last_bwd[j], op);
                            fused_dc = true;
                            break;
                        }
                        if (direct) {
                            d.epi.dst[d.epi.ndst++] = d0.slots[k] + so * Q * d0.slot_ld;
                            d.epi.ldd = static_cast<long long>(Q) * d0.slot_ld;
                        } else {
                            d.epi.dst[d.epi.ndst++] = wl.dcols + so * drows * wl.ldk;
                            d.epi.ldd = wl.ldk;
                        }
                        prepare(d, wl.p_dgrad[j], w.gpu);
                        fl = li.dense_conv ? 2.0 * rows * pix * wl.u * Q * li.in_units
                                           : 2.0 * rows * li.H * li.W * li.in_units * li.ksz * li.ksz * wl.u;
                        int op = add_op(w.gpu, w.sb, gemm_launch(&wl.p_dgrad[j], &wl.d_dgrad[j], w.sb), wl.delta_ready[j],
                                        nk(wl.p_dgrad[j]), OP_DGRAD_GEMM, fl);
                        wl.dgrad_op[j] = op;
                        const float* dc = wl.dcols + so * drows * wl.ldk;
                        const bool dcv = li.dense_conv;
                        const long long ldk = dcv ? li.in_units : wl.ldk;  // dense conv: pixel-major [img*Q][C]
                        const int H = li.H, W = li.W, C = li.in_units, ks = dcv ? 1 : li.ksz, pd = dcv ? 0 : li.pad,
                                  strd = li.stride;
                        if (c2m) {
                            c2m_src.dcols = dc;
                            c2m_src.ldk = ldk;
                            c2m_src.C = C;
                            c2m_src.p = pd;
                            c2m_src.Ho = li.Ho();
                            c2m_src.Wo = li.Wo();
                            c2m_src.c0 = workers_[dests[0]]->at(l - 1).lo;
                        }
                        for (int di : direct || c2m ? std::vector<int>{} : dests) {
                            WLayer& dl = workers_[di]->at(l - 1);
                            float* dst = dl.slots[k] + so * H * W * dl.slot_ld;
                            const long long ldo = dl.slot_ld;
                            const int c0 = dl.lo, nc = dl.u;
                            cudaStream_t st = w.sb;
                            op = add_op(w.gpu, st, [=]() {
                                return launch_col2im(dc, ldk, rows, H, W, C, ks, pd, c0, nc, dst, ldo, st, strd);
                            }, {op}, 1, OP_CONV_MERGE);
                        }
                        w.last_bwd[j] = std::max(w.last_bwd[j], op);
                        dgrad_ops.push_back(op);
                        continue;
                    }
                    if (li.kind == 1) {
                        ConvShape cs;
                        cs.N = rows;
                        cs.H = li.H;
                        cs.W = li.W;
                        cs.C = li.in_units;
                        cs.ksz = li.ksz;
                        cs.pad = li.pad;
                        cs.u = wl.u;
                        d = conv_dgrad_desc(cs, wl.delta + so * wl.delta_img, wl.ldd, wl.W);
                        fl = 2.0 * rows * li.H * li.W * li.in_units * li.ksz * li.ksz * wl.u;
                        rows_per_img = static_cast<long long>(li.H) * li.W;
                    } else {
                        d.a = Operand{wl.delta + so * wl.ldd, rows, wl.u, wl.ldd, false};
                        d.b = Operand{wl.W, wl.u, fi, wl.ldw, true};
                        d.M = rows;
                        d.N = fi;
                        d.K = wl.u;
                        fl = 2.0 * rows * wl.u * fi;
                        rows_per_img = 1;
                    }
                    d.epi = EpiParams{};
                    d.epi.mode = EPI_SLOTS;
                    const int scale = li.kind == 1 ? 1 : hw;
                    for (int di : dests) {
                        WLayer& dl = workers_[di]->at(l - 1);
                        const int sg = d.epi.nseg++;
                        d.epi.seg_lo[sg] = dl.lo * scale;
                        d.epi.seg_hi[sg] = dl.hi * scale;
                        d.epi.seg_ld[sg] = dl.slot_ld;
                        d.epi.seg_dst[sg] = dl.slots[k] + so * rows_per_img * dl.slot_ld;
                    }
                    prepare(d, wl.p_dgrad[j], w.gpu);
                    const int op = add_op(w.gpu, w.sb, gemm_launch(&wl.p_dgrad[j], &wl.d_dgrad[j], w.sb),
                                          wl.delta_ready[j], nk(wl.p_dgrad[j]), OP_DGRAD_GEMM, fl);
                    wl.dgrad_op[j] = op;
                    w.last_bwd[j] = std::max(w.last_bwd[j], op);
                    dgrad_ops.push_back(op);
                }
                if (fused_dc) continue;
                for (int di : dests) {
                    Worker& dw = *workers_[di];
                    WLayer& dl = dw.at(l - 1);
                    ConvMerge cm;
                    const long long rows_per_img = li.kind == 1 ? hw : 1;
                    for (float* sp : dl.slots) cm.slots.slot[cm.slots.n++] = sp + so * rows_per_img * dl.slot_ld;
                    // a dense consumer's CHW-flatten slot over a 1 x 1 pooled grid is
                    // the pixel-major layout (vectorised merge kernel)
                    cm.slot_kind = (li.kind == 1 || lb.Hq() * lb.Wq() == 1) ? 0 : 1;
                    cm.lds = dl.slot_ld;
                    cm.imgs = rows;
                    cm.Ho = lb.Ho();
                    cm.Wo = lb.Wo();
                    cm.uch = dl.u;
                    cm.pool = lb.pool;
                    cm.argmax = dl.argmax ? dl.argmax + so * hw * dl.u : nullptr;
                    if (relu_below) {
                        if (dl.U != nullptr && dl.u_written) {
                            cm.mask_kind = 1;
                            cm.U = dl.U + so * lb.Ho() * lb.Wo() * dl.ldu;
                            cm.ldu = dl.ldu;
                        } else {
                            // pooled layers whose pre-pool rows were never stored (pool fused
                            // across warp pairs) mask at the pooled pixel
                            cm.mask_kind = lb.pool == 2 ? 3 : 2;
                            cm.act = act_buf(dw.gpu, l - 1) + aoff(l - 1, j) * img_elems(l - 1);
                            cm.act_layout = lay_[l - 1];
                            cm.act_layout.col0 = dl.lo;
                        }
                    }
                    cm.d_pad = dl.delta + so * dl.delta_img;
                    cm.q = lb.dq();
                    cm.ldd = dl.ldd;
                    cudaStream_t st = dw.sb;
                    float* dbp = dl.partial + static_cast<long long>(j) * conv_merge_blocks() * dl.u;
                    int op;
                    if (res_dest) {
                        // average-pool routing and / or the shortcut term of the residual
                        // layer reading this layer's output (added before the ReLU mask)
                        SkipGrad sg;
                        std::vector<int> mdeps = dgrad_ops;
                        if (const int r = res_consumer(l - 1)) {
                            const LayerInfo& lr = net_.info[r - 1];
                            WLayer* src = nullptr;
                            for (int wi : layer_workers_[r]) {
                                WLayer& cand = workers_[wi]->at(r);
                                if (cand.contributor && cand.lo <= dl.lo && dl.hi <= cand.hi) src = &cand;
                            }
                            if (src == nullptr)
                                throw std::invalid_argument("layers " + S(l - 1) + "," + S(r) +
                                                            ": residual shortcut crosses shard boundaries");
                            sg.d = src->delta + so * src->delta_img;
                            sg.ldd = src->ldd;
                            sg.q = lr.dq();
                            sg.hq = lr.Ho() + 2 * sg.q;
                            sg.wq = lr.Wo() + 2 * sg.q;
                            sg.f = lb.Hq() / lr.Ho();
                            sg.c0 = dl.lo - src->lo;
                            mdeps.insert(mdeps.end(), src->delta_ready[j].begin(), src->delta_ready[j].end());
                        }
                        const int pavg = lb.pool_avg;
                        if (c2m) {
                            const Col2imSrc cx = c2m_src;
                            op = add_op(dw.gpu, st, [=]() { return launch_conv_merge_res_col2im(cm, pavg, sg, cx, dbp, st); },
                                        mdeps, 1, OP_CONV_MERGE);
                        } else {
                            op = add_op(dw.gpu, st, [=]() { return launch_conv_merge_res(cm, pavg, sg, dbp, st); }, mdeps, 1,
                                        OP_CONV_MERGE);
                        }
                    } else {
                        op = add_op(dw.gpu, st, [=]() { return launch_conv_merge(cm, dbp, st); }, dgrad_ops, 1,
                                    OP_CONV_MERGE);
                    }
                    dl.delta_ready[j] = {op};
                    dw.last_bwd[j] = std::max(dw.last_bwd[j], op);
                }
                continue;
            }
            for (size_t k = 0; k < contrib.size(); ++k) {
                Worker& w = *workers_[contrib[k]];
                WLayer& wl = w.at(l);
                GemmDesc& d = wl.d_dgrad[j];
                d.a = Operand{wl.delta + so * wl.ldd, rows, wl.u, wl.ldd, false};
                d.b = Operand{wl.W, wl.u, fi, wl.ldw, true};
                d.M = rows;
                d.N = fi;
                d.K = wl.u;
                d.epi = EpiParams{};
                d.epi.mode = EPI_SLOTS;
                const bool ncl = nccl_layer(l - 1);
                for (int di : dests) {
                    Worker& dw = *workers_[di];
                    WLayer& dl = dw.at(l - 1);
                    const int s = d.epi.nseg++;
                    d.epi.seg_lo[s] = dl.lo;
                    d.epi.seg_hi[s] = dl.hi;
                    d.epi.seg_ld[s] = dl.ldd;
                    if (ncl) {  // NCCL backend: block s of the packed per-rank partial [g][rows][u]
                        const long long gsz = static_cast<long long>(dests.size());
                        d.epi.seg_ld[s] = dl.u;
                        d.epi.seg_dst[s] = wl.rs_send + so * gsz * dl.u + static_cast<long long>(s) * rows * dl.u;
                    } else if (single) {
                        d.epi.seg_dst[s] = dl.delta + so * dl.ldd;
                        if (relu_below) {
                            d.epi.seg_mask[s] = act_buf(dw.gpu, l - 1) + so * ld_of(fi);
                            d.epi.seg_mask_ld[s] = ld_of(fi);
                        }
                    } else {
                        d.epi.seg_dst[s] = dl.slots[k] + so * dl.ldd;
                    }
                }
                prepare(d, wl.p_dgrad[j], w.gpu);
                const int op = add_op(w.gpu, w.sb, gemm_launch(&wl.p_dgrad[j], &wl.d_dgrad[j], w.sb),
                                      wl.delta_ready[j], nk(wl.p_dgrad[j]), OP_DGRAD_GEMM, 2.0 * rows * wl.u * fi);
                wl.dgrad_op[j] = op;
                w.last_bwd[j] = std::max(w.last_bwd[j], op);
                dgrad_ops.push_back(op);
            }
            int rs_op = -1;
            if (nccl_layer(l - 1)) {
                // ncclReduceScatter: rank k receives the sum over contributors of
                // block k (its own columns), on each worker's input-gradient stream
                std::vector<const float*> snd;
                std::vector<float*> rcv;
                std::vector<cudaStream_t> sts;
                const long long gsz = static_cast<long long>(dests.size());
                for (size_t k = 0; k < contrib.size(); ++k) {
                    Worker& w = *workers_[contrib[k]];
                    WLayer& dl = workers_[dests[k]]->at(l - 1);
                    snd.push_back(w.at(l).rs_send + so * gsz * dl.u);
                    rcv.push_back(dl.rs_recv + so * dl.u);
                    sts.push_back(w.sb);
                }
                const NcclGroup* grp = nccl_[module_index(l - 1) - 1].get();
                const int ud = workers_[dests.front()]->at(l - 1).u;
                Worker& w0 = *workers_[contrib.front()];
                rs_op = add_op(w0.gpu, w0.sb, [=]() { return nccl_reduce_scatter(*grp, snd, rcv, rows, ud, sts); },
                               dgrad_ops, 0, OP_REDUCE);
            }
            for (int di : dests) {
                Worker& dw = *workers_[di];
                WLayer& dl = dw.at(l - 1);
                if (rs_op >= 0) {  // the reduced block -> mask -> delta
                    ReduceSlots rs;
                    rs.slot[rs.n++] = dl.rs_recv + so * dl.u;
                    const float* mask = relu_below ? act_buf(dw.gpu, l - 1) + so * ld_of(fi) + dl.lo : nullptr;
                    const long long ldm = ld_of(fi), lds = dl.u, ldd = dl.ldd;
                    float* out = dl.delta + so * dl.ldd;
                    const int u = dl.u;
                    cudaStream_t st = dw.sb;
                    const int op = add_op(dw.gpu, st, [=]() {
                        return launch_reduce_mask(rs, lds, rows, u, mask, ldm, out, ldd, st);
                    }, {rs_op}, 1, OP_REDUCE);
                    dl.delta_ready[j] = {op};
                    dw.last_bwd[j] = std::max(dw.last_bwd[j], op);
                    continue;
                }
                if (single) {
                    dl.delta_ready[j] = dgrad_ops;
                    dw.last_bwd[j] = std::max(dw.last_bwd[j], dgrad_ops.front());
                    continue;
                }
                ReduceSlots rs;
                for (float* sp : dl.slots) rs.slot[rs.n++] = sp + so * dl.ldd;
                const float* mask = relu_below ? act_buf(dw.gpu, l - 1) + so * ld_of(fi) + dl.lo : nullptr;
                const long long ldm = ld_of(fi);
                float* out = dl.delta + so * dl.ldd;
                const long long ldd = dl.ldd;
                const int u = dl.u;
                cudaStream_t s = dw.sb;
                const int op = add_op(dw.gpu, s, [=]() {
                    return launch_reduce_mask(rs, ldd, rows, u, mask, ldm, out, ldd, s);
                }, dgrad_ops, 1, OP_REDUCE);
                dl.delta_ready[j] = {op};
                dw.last_bwd[j] = std::max(dw.last_bwd[j], op);
            }
        }
        // module-1 / layer-1 workers: their backward ends when delta_1 is ready
        for (int wi : layer_workers_[1])
            for (int op : workers_[wi]->at(1).delta_ready[j])
                workers_[wi]->last_bwd[j] = std::max(workers_[wi]->last_bwd[j], op);
        if (per_mb_wgrad_) per_mb_wgrads(j, first_op);
    };

    // interleave creation so every dependency already exists: F(1..gate), then
    // B(j-gate) before F(j) (the pipelined order, schedule.cpp:254-329)
    const int gate = cfg_.gate > 0 ? cfg_.gate : m;
    for (int k = 0; k < m + gate; ++k) {
        if (k - gate >= 0 && k - gate < m) backward(k - gate);
        if (k < m) forward(k);
    }

    // ---------------- updates (train_partitioned.cpp:632-651)
    cur_mb_ = -1;
    int bwd_join = -1;
    if (cfg_.mode == 1) {
        std::vector<int> all;
        for (auto& wp : workers_)
            for (WLayer& wl : wp->layers) {
                for (int j = 0; j < m; ++j) {
                    all.insert(all.end(), wl.delta_ready[j].begin(), wl.delta_ready[j].end());
                    if (wl.dgrad_op[j] >= 0) all.push_back(wl.dgrad_op[j]);
                }
            }
        bwd_join = add_op(g0.ordinal, g0.main, nullptr, all, 0);  // std::barrier (:633)
    }
    const float inv_b = 1.f / static_cast<float>(cfg_.batch);
    static const bool no_side = dev_knob("PPB_NO_SIDE_JOB");
    // proposed policy: the layer's update = one reduction over the m x
    // acc_slices partial slices (micro-batch order, then split order) applying
    // the real epilogue (SGD on W with the bias update in the same launch, or
    // dWx for a dense-conv layer, then its fold + SGD)
    auto reduce_update = [&](Worker& w, WLayer& wl, int join) {
        Gpu& g = gpu_of(w.gpu);
        const LayerInfo& li = net_.info[wl.layer - 1];
        std::vector<int> deps = wl.wg_op;
        for (int j = 0; j < m; ++j) {
            deps.insert(deps.end(), wl.delta_ready[j].begin(), wl.delta_ready[j].end());
            if (wl.dgrad_op[j] >= 0) deps.push_back(wl.dgrad_op[j]);  // dgrads read W
        }
        if (join >= 0) deps.push_back(join);
        const bool fm = bias_from_merge(wl);
        const int chunks = fm ? cfg_.m * conv_merge_blocks() * wl.db_q : cfg_.m * wl.cc_mb;
        wl.p_red = wl.p_wg[0];
        wl.p_red.sk.ws = wl.acc_ws;
        wl.p_red.sk.splits = m * wl.acc_slices;
        wl.p_red.sk.partial = 0;
        wl.p_red.sk.deferred = 0;
        wl.p_red.sk.fixup = 0;
        wl.p_red.epi = wl.d_wg[0].epi;
        wl.p_red.epi.M = wl.p_red.M;
        wl.p_red.epi.N = wl.p_red.N;
        cudaStream_t s = w.su;
        const double* alpha = &g.st->alpha;
        if (!li.dense_conv) {
            wl.p_red.sk.bpart = wl.partial;
            wl.p_red.sk.bias = wl.bias;
            wl.p_red.sk.bchunks = chunks;
            wl.p_red.sk.bu = wl.u;
            const TcGemmPlan* pr = &wl.p_red;
            add_op(w.gpu, s, [pr, s]() { return tc_gemm_launch_reduce(*pr, s); }, deps, 1, OP_BIAS);
            return;
        }
        const TcGemmPlan* pr = &wl.p_red;
        const int rop = add_op(w.gpu, s, [pr, s]() { return tc_gemm_launch_reduce(*pr, s); }, deps, 1, OP_BIAS);
        const DenseConvGeom dg = wl.dcg;
        const float* dWx = wl.dWx;
        float* Wp = wl.W;
        float* Wx = wl.Wx;
        int* flag = &g.st->diverge_flag;
        const float* bp = wl.partial;
        float* bb = wl.bias;
        add_op(w.gpu, s, [=]() { return launch_dense_conv_fold_sgd(dg, dWx, Wp, Wx, alpha, inv_b, flag, s, bp, chunks, bb); },
               {rop}, 1, OP_BIAS);
    };
    for (auto& wp : workers_) {
        Worker& w = *wp;
        Gpu& g = gpu_of(w.gpu);
        // wgrads in backward order (top layer first: each can start as soon as
        // its delta exists); a split-K wgrad's reduction + SGD is carried by the
        // next wgrad GEMM on the stream (SideJob) instead of its own kernel
        // pending side job: the previous split-K wgrad's reduction, or the
        // previous dense-conv layer's weight update (its op is then a no-op)
        // two weight-gradient streams (alternate layers) so independent wgrads of
        // the bottom layers -- which all become ready at the end of the dgrad
        // chain -- overlap instead of queueing; each stream keeps its own
        // side-job chain
        static const bool two_su = wgrad_two_streams();
        struct Chain {
            TcGemmPlan* prev_plan = nullptr;
            WLayer* prev_wl = nullptr;
            int prev_op = -1;
            SideJob pend_fold;
            bool* pend_flag = nullptr;
            int pend_fold_op = -1;
        } chains[2];
        int ci = 0;  // chain of the layer being built
        WLayer* cur_wl = nullptr;
        auto link_side = [&](TcGemmPlan* p, int op, bool carrier_ok) {
            TcGemmPlan*& prev_plan = chains[ci].prev_plan;
            WLayer*& prev_wl = chains[ci].prev_wl;
            int& prev_op = chains[ci].prev_op;
            SideJob& pend_fold = chains[ci].pend_fold;
            bool*& pend_flag = chains[ci].pend_flag;
            int& pend_fold_op = chains[ci].pend_fold_op;
            if (!tf32) return;
            const bool can = carrier_ok && !no_side && (p->halo == 0 || p->halo == 2);  // halo wgrads carry too
            if (pend_flag != nullptr) {
                if (can) {
                    p->sj = pend_fold;
                    *pend_flag = true;
                    ops_[pend_fold_op].kernels -= 1;
                }
            } else if (prev_plan != nullptr && can && prev_plan->sk.splits > 1 && !prev_plan->sk.fixup &&
                       !prev_plan->sk.deferred &&
                       !(prev_wl != nullptr && net_.info[prev_wl->layer - 1].dense_conv)) {  // its fold reads dWx
                p->sj.on = 1;
                static const bool side_scalar = dev_knob("PPB_SIDE_SCALAR");
                p->sj.scalar = side_scalar ? 1 : 0;
                p->sj.M = prev_plan->M;
                p->sj.N = prev_plan->N;
                p->sj.sk = prev_plan->sk;
                p->sj.epi = prev_plan->epi;
                prev_plan->sk.deferred = 1;
                ops_[prev_op].kernels -= 1;
                // the deferred GEMM now writes only its split-K workspace: it no
                // longer waits for its layer's dgrad (which reads W); the update
                // rides in this GEMM, which follows that dgrad through its own
                // error signal (produced after it)
                // opt-in (DEV builds, PPB_WGRAD_EARLY=1): measured equal on the VGG-16 step
                // (2.303 vs 2.306 ms, 3 A/B pairs): the early wgrad only contends with
                // the dgrad for L2 bandwidth
                static const bool strict = !dev_knob("PPB_WGRAD_EARLY");
                if (prev_wl != nullptr && !strict) {
                    auto& dv = ops_[prev_op].deps;
                    for (int dg : prev_wl->dgrad_op)
                        if (dg >= 0) dv.erase(std::remove(dv.begin(), dv.end(), dg), dv.end());
                }
            }
            pend_flag = nullptr;
            prev_plan = p;
            prev_op = op;
            prev_wl = cur_wl;
        };
        for (auto wit = w.layers.rbegin(); wit != w.layers.rend(); ++wit) {
            WLayer& wl = *wit;
            const int l = wl.layer;
            cur_layer_ = l;
            const LayerInfo& li = net_.info[l - 1];
            GemmDesc& d = wl.d_wgrad;
            double wfl;
            long long bias_rows;
            wgrad_desc(w, wl, -1, d, &wfl, &bias_rows);
            if (per_mb_wgrad_) {  // proposed policy: one reduction (+ SGD / dWx) over the micro-batch slices
                reduce_update(w, wl, bwd_join);
                continue;
            }
            prepare(d, wl.p_wgrad, w.gpu);
            std::vector<int> deps;
            for (int j = 0; j < m; ++j) {
                deps.insert(deps.end(), wl.delta_ready[j].begin(), wl.delta_ready[j].end());
                if (wl.dgrad_op[j] >= 0) deps.push_back(wl.dgrad_op[j]);
            }
            if (bwd_join >= 0) deps.push_back(bwd_join);
            ci = two_su ? (l & 1) : 0;
            cur_wl = &wl;
            cudaStream_t s = ci ? w.su2 : w.su;
            SideJob& pend_fold = chains[ci].pend_fold;
            bool*& pend_flag = chains[ci].pend_flag;
            int& pend_fold_op = chains[ci].pend_fold_op;
            const float* delta = wl.delta;
            const long long ldd = wl.ldd;
            const int b = static_cast<int>(bias_rows), u = wl.u;
            float* partial = wl.partial;
            float* bias = wl.bias;
            const double* alpha = &g.st->alpha;
            // conv: db partials came with the merges (conv_merge or the EPI_MERGE epilogue)
            const bool from_merge = li.kind == 1 && !wl.db_colsum;
            const int chunks = cfg_.m * conv_merge_blocks() * wl.db_q;
            const int splits = tf32 ? wl.p_wgrad.sk.splits : 1;
            if (li.dense_conv) {
                // dWx GEMM, then one launch: fold + SGD on W + re-expand Wx (+ the
                // bias update from the merge partials)
                std::vector<int> gdeps = deps;
                if (!from_merge)
                    gdeps = {add_op(w.gpu, s, [=]() {
                        return launch_bias_update(delta, ldd, b, u, partial, bias, alpha, inv_b, s);
                    }, deps, 2, OP_BIAS)};
                const int gop = add_op(w.gpu, s, gemm_launch(&wl.p_wgrad, &wl.d_wgrad, s), gdeps, nk(wl.p_wgrad),
                                       OP_WGRAD_GEMM, wfl);
                link_side(&wl.p_wgrad, gop, true);
                const DenseConvGeom dg = wl.dcg;
                const float* dWx = wl.dWx;
                float* Wp = wl.W;
                float* Wx = wl.Wx;
                int* flag = &g.st->diverge_flag;
                const float* bp = from_merge ? partial : nullptr;
                float* bb = from_merge ? bias : nullptr;
                bool* deferred = &wl.fold_deferred;
                const int fop = add_op(w.gpu, s, [=]() {
                    if (*deferred) return cudaSuccess;  // carried by the next wgrad GEMM (SideJob)
                    return launch_dense_conv_fold_sgd(dg, dWx, Wp, Wx, alpha, inv_b, flag, s, bp, chunks, bb);
                }, {gop}, 1, OP_BIAS);
                // carrying the update in the next wgrad GEMM measured slower (2.287
                // vs 2.281 ms: its 51 MB of traffic slows that GEMM's mainloop more
                // than the low-priority kernel costs), so it is opt-in
                const bool fold_side = dev_knob("PPB_FOLD_SIDE");
                if (tf32 && dense_conv_is_2x2(dg) && fold_side) {  // offer the update to the next wgrad GEMM
                    SideJob& f = pend_fold;
                    f = SideJob{};
                    f.on = 1;
                    f.kind = 1;
                    f.dWx = dWx;
                    f.Wm = Wp;
                    f.Wx = Wx;
                    f.dc_u = dg.u;
                    f.dc_C = dg.C;
                    f.dc_ck = dg.ck;
                    f.dc_ldw = dg.ldw;
                    f.dc_ldx = dg.ldx;
                    f.epi.alpha = alpha;
                    f.epi.inv_b = inv_b;
                    f.epi.flag = flag;
                    f.sk.bpart = bp;
                    f.sk.bias = bb;
                    f.sk.bchunks = chunks;
                    f.sk.bu = u;
                    pend_flag = deferred;
                    pend_fold_op = fop;
                }
                continue;
            }
            if (from_merge && splits > 1 && !wl.p_wgrad.sk.fixup) {
                // the bias update rides in the wgrad's split-K reduction launch
                wl.p_wgrad.sk.bpart = partial;
                wl.p_wgrad.sk.bias = bias;
                wl.p_wgrad.sk.bchunks = chunks;
                wl.p_wgrad.sk.bu = u;
                const int gop = add_op(w.gpu, s, gemm_launch(&wl.p_wgrad, &wl.d_wgrad, s), deps, 2, OP_WGRAD_GEMM, wfl);
                link_side(&wl.p_wgrad, gop, true);
                continue;
            }
            const int bop = add_op(w.gpu, s, [=]() {
                if (from_merge) return launch_bias_from_partials(partial, chunks, u, bias, alpha, inv_b, s);
                return launch_bias_update(delta, ldd, b, u, partial, bias, alpha, inv_b, s);
            }, deps, from_merge ? 1 : 2, OP_BIAS);
            const int gop = add_op(w.gpu, s, gemm_launch(&wl.p_wgrad, &wl.d_wgrad, s), {bop}, nk(wl.p_wgrad),
                                   OP_WGRAD_GEMM, wfl);
            link_side(&wl.p_wgrad, gop, true);
        }
        // the last split-K wgrad of each stream has no carrier: its GEMM still
        // runs as soon as its error signal exists (concurrently with its own
        // layer's dgrad, which reads W) and the reduction + update follows both
        // opt-in (DEV builds, PPB_WGRAD_EARLY=1): measured equal on the VGG-16 step
                // (2.303 vs 2.306 ms, 3 A/B pairs): the early wgrad only contends with
                // the dgrad for L2 bandwidth
                static const bool strict = !dev_knob("PPB_WGRAD_EARLY");
        for (Chain& c : chains) {
            TcGemmPlan* pp = c.prev_plan;
            if (strict || !tf32 || pp == nullptr || c.prev_wl == nullptr || pp->sk.splits <= 1 || pp->sk.fixup ||
                pp->sk.deferred || net_.info[c.prev_wl->layer - 1].dense_conv)
                continue;
            pp->sk.deferred = 1;
            ops_[c.prev_op].kernels -= 1;
            auto& dv = ops_[c.prev_op].deps;
            std::vector<int> rdeps{c.prev_op};
            for (int dg : c.prev_wl->dgrad_op)
                if (dg >= 0) {
                    dv.erase(std::remove(dv.begin(), dv.end(), dg), dv.end());
                    rdeps.push_back(dg);
                }
            cur_layer_ = c.prev_wl->layer;
            cudaStream_t s = ops_[c.prev_op].stream;
            add_op(w.gpu, s, [pp, s]() { return tc_gemm_launch_reduce(*pp, s); }, rdeps, 1, OP_BIAS);
        }
    }

    // ---------------- finalize per GPU, then the iteration join
    std::vector<int> finals;
    for (auto& gp : gpus_) {
        Gpu& g = *gp;
        std::map<cudaStream_t, int> last;
        for (int i = 0; i < static_cast<int>(ops_.size()); ++i)
            if (ops_[i].gpu == g.ordinal) last[ops_[i].stream] = i;
        std::vector<int> deps;
        for (auto& kv : last) deps.push_back(kv.second);
        StepState* st = g.st;
        const double* lr = g.loss_row;
        const int* cr = g.correct_row;
        double* lh = g.loss_hist;
        double* ah = g.acc_hist;
        const int b = cfg_.batch, cap = hist_cap_;
        const int write = g.ordinal == main_gpu_;
        cudaStream_t s = g.main;
        finals.push_back(add_op(g.ordinal, s, [=]() {
            return launch_finalize(st, lr, cr, b, lh, ah, cap, write, s);
        }, deps, 1, OP_FINALIZE));
    }
    {
        std::map<cudaStream_t, int> last;
        for (int i = 0; i < static_cast<int>(ops_.size()); ++i) last[ops_[i].stream] = i;
        std::vector<int> deps = finals;
        for (auto& kv : last) deps.push_back(kv.second);
        end_op_ = add_op(g0.ordinal, g0.main, nullptr, deps, 0);
    }
    kernels_per_step_ = 0;
    for (const Op& op : ops_) kernels_per_step_ += op.kernels;
    (void)F;
}

void Session::enqueue_iteration() {
    std::set<cudaStream_t> joined;
    for (int i = 0; i < static_cast<int>(ops_.size()); ++i) {
        Op& op = ops_[i];
        check(cudaSetDevice(op.gpu), "cudaSetDevice");
        if (i != begin_op_ && !joined.count(op.stream) && op.stream != ops_[begin_op_].stream)
            check(cudaStreamWaitEvent(op.stream, ops_[begin_op_].ev, 0), "fork");
        joined.insert(op.stream);
        for (int d : op.deps)
            if (ops_[d].stream != op.stream) check(cudaStreamWaitEvent(op.stream, ops_[d].ev, 0), "wait");
        if (op.launch) check(op.launch(), "kernel launch");
        check(cudaEventRecord(op.ev, op.stream), "record");
    }
}

void Session::enqueue_iteration_timed(std::vector<cudaEvent_t>& t0, std::vector<cudaEvent_t>& t1) {
    std::set<cudaStream_t> joined;
    if (!serialise_) {
        // concurrent timeline: hold the step behind a spin so every launch is
        // queued before the first kernel runs (as in the graph), then let the
        // streams overlap; events record each op's start / end
        check(cudaSetDevice(ops_[begin_op_].gpu), "cudaSetDevice");
        check(launch_spin(3000000, ops_[begin_op_].stream), "spin");
    }
    for (int i = 0; i < static_cast<int>(ops_.size()); ++i) {
        Op& op = ops_[i];
        check(cudaSetDevice(op.gpu), "cudaSetDevice");
        if (i != begin_op_ && !joined.count(op.stream) && op.stream != ops_[begin_op_].stream)
            check(cudaStreamWaitEvent(op.stream, ops_[begin_op_].ev, 0), "fork");
        joined.insert(op.stream);
        for (int d : op.deps)
            if (ops_[d].stream != op.stream) check(cudaStreamWaitEvent(op.stream, ops_[d].ev, 0), "wait");
        if (op.launch) {
            if (serialise_) check(launch_spin(30000, op.stream), "spin");  // absorbs the launch latency of what follows
            check(cudaEventRecord(t0[i], op.stream), "record");
            check(op.launch(), "kernel launch");
            check(cudaEventRecord(t1[i], op.stream), "record");
            // serialised: every op runs alone, so its CUDA-event duration is the
            // kernel's own time (the graph overlaps streams; events cannot
            // separate concurrent kernels)
            if (serialise_) check(cudaEventSynchronize(t1[i]), "serialise");
        }
        check(cudaEventRecord(op.ev, op.stream), "record");
    }
}

float Session::time_steps(int iterations) {
    Gpu& g0 = *gpus_[0];
    check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
    cudaEvent_t a, b;
    check(cudaEventCreate(&a), "event");
    check(cudaEventCreate(&b), "event");
    check(cudaEventRecord(a, g0.main), "record");
    step(iterations);
    check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
    check(cudaEventRecord(b, g0.main), "record");
    check(cudaEventSynchronize(b), "sync");
    float ms = 0.f;
    check(cudaEventElapsedTime(&ms, a, b), "elapsed");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    sync();
    return ms;
}

void Session::profile(int iterations, double* ms, int* count, double* flops, int nkinds) {
    const int n = static_cast<int>(ops_.size());
    std::vector<cudaEvent_t> t0(n, nullptr), t1(n, nullptr);
    for (int i = 0; i < n; ++i) {
        if (!ops_[i].launch) continue;
        check(cudaSetDevice(ops_[i].gpu), "cudaSetDevice");
        check(cudaEventCreate(&t0[i]), "event");
        check(cudaEventCreate(&t1[i]), "event");
    }
    for (int k = 0; k < nkinds; ++k) {
        ms[k] = 0;
        count[k] = 0;
        flops[k] = 0;
    }
    last_op_ms_.assign(n, 0.0);
    last_op_start_.assign(n, 0.0);
    for (int it = 0; it < iterations; ++it) {
        enqueue_iteration_timed(t0, t1);
        ++steps_enqueued_;
        Gpu& g0 = *gpus_[0];
        check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
        check(cudaEventRecord(g0.ev_done, g0.main), "record");
        sync();
        for (int i = 0; i < n; ++i) {
            if (!ops_[i].launch || ops_[i].kind >= nkinds) continue;
            float e = 0.f;
            check(cudaEventElapsedTime(&e, t0[i], t1[i]), "elapsed");
            last_op_ms_[i] += e;
            int first = -1;
            for (int f = 0; f < n && first < 0; ++f)
                if (ops_[f].launch && ops_[f].gpu == ops_[i].gpu) first = f;
            float st = 0.f;
            if (first >= 0) check(cudaEventElapsedTime(&st, t0[first], t0[i]), "elapsed");
            last_op_start_[i] = st;
            ms[ops_[i].kind] += e;
            count[ops_[i].kind] += 1;
            flops[ops_[i].kind] += ops_[i].flops;
        }
    }
    for (int i = 0; i < n; ++i) {
        if (t0[i]) cudaEventDestroy(t0[i]);
        if (t1[i]) cudaEventDestroy(t1[i]);
    }
}

int Session::profile_ops(int* kind, int* layer, int* info, double* ms, double* flops, int cap) {
    int k = 0;
    for (int i = 0; i < static_cast<int>(ops_.size()) && i < static_cast<int>(last_op_ms_.size()); ++i) {
        if (!ops_[i].launch) continue;
        if (k < cap) {
            kind[k] = ops_[i].kind;
            layer[k] = ops_[i].layer;
            info[k] = ops_[i].info;
            ms[k] = last_op_ms_[i];
            flops[k] = ops_[i].flops;
        }
        ++k;
    }
    return k;
}

int Session::op_meta(int* mb, int* device, int* role, int cap) {
    std::map<cudaStream_t, std::pair<int, int>> who;  // stream -> (plan device, role)
    for (const auto& w : workers_) {
        who[w->sf] = {w->device, 0};
        who[w->sb] = {w->device, 1};
        who[w->su] = {w->device, 2};
        who[w->su2] = {w->device, 2};
    }
    int k = 0;
    for (int i = 0; i < static_cast<int>(ops_.size()); ++i) {
        if (!ops_[i].launch) continue;
        if (k < cap) {
            auto it = who.find(ops_[i].stream);
            mb[k] = ops_[i].mb;
            device[k] = it == who.end() ? 0 : it->second.first;
            role[k] = it == who.end() ? 3 : it->second.second;
        }
        ++k;
    }
    return k;
}

int Session::profile_starts(double* start_ms, int* stream_id, int cap) {
    std::map<cudaStream_t, int> ids;
    int k = 0;
    for (int i = 0; i < static_cast<int>(ops_.size()) && i < static_cast<int>(last_op_start_.size()); ++i) {
        if (!ops_[i].launch) continue;
        if (!ids.count(ops_[i].stream)) {
            const int id = static_cast<int>(ids.size());
            ids[ops_[i].stream] = id;
        }
        if (k < cap) {
            start_ms[k] = last_op_start_[i];
            stream_id[k] = ids[ops_[i].stream];
        }
        ++k;
    }
    return k;
}

void Session::capture_graph() {
    Gpu& g0 = *gpus_[0];
    check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
    if (cudaStreamBeginCapture(g0.main, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    bool ok = true;
    try {
        enqueue_iteration();
    } catch (...) {
        ok = false;
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(g0.main, &graph);
    if (!ok || e != cudaSuccess || graph == nullptr) {
        cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        return;
    }
    if (cudaGraphInstantiate(&graph_exec_, graph, 0) != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(graph);
        graph_exec_ = nullptr;
        return;
    }
    graph_ = graph;
    graph_ok_ = true;
}

// ------------------------------------------------------------------ runtime

void Session::validate_labels(const int* labels) const {
    const int L = net_.L();
    const int F = net_.dims[L];
    for (int i = 0; i < cfg_.batch; ++i) {
        const int y = labels[i];
        if (cfg_.loss == 1 && (y < 0 || y >= F)) throw std::invalid_argument("label out of range");
        if (cfg_.loss == 0 && F > 1 && (y < 0 || y >= F))
            throw std::invalid_argument("label out of range for one-hot target");
    }
}

void Session::load_batch(const double* X64, const float* X32, const int* labels) {
    stage_batch(X64, X32, labels, 0);
    convert_staged(0, X64 != nullptr);
}

// Phase 1 of a batch load: the host batch (fp64 or fp32 rows, as given) and
// its labels into device staging slot k on each GPU's copy stream, once the
// batch that used slot k before has been converted out of it.
void Session::stage_batch(const double* X64, const float* X32, const int* labels, int k) {
    validate_labels(labels);
    // accuracy() accepts binary labels only (tinynet.cpp:376-378); the
    // reference raises it from the history collector after the workers
    // finished, so it is reported by sync() after any divergence error.
    pending_acc_error_ = false;
    if (!cfg_.multiclass)
        for (int i = 0; i < cfg_.batch; ++i)
            if (labels[i] != 0 && labels[i] != 1) pending_acc_error_ = true;
    const size_t n = static_cast<size_t>(cfg_.batch) * net_.dims[0];
    for (auto& gp : gpus_) {
        Gpu& g = *gp;
        check(cudaSetDevice(g.ordinal), "cudaSetDevice");
        check(cudaStreamWaitEvent(g.copy, g.ev_consumed[k], 0), "wait");
        if (g.needs_x) {
            void* dst = k ? g.xstage2 : g.xstage;
            if (X64 != nullptr) check(cudaMemcpyAsync(dst, X64, sizeof(double) * n, cudaMemcpyHostToDevice, g.copy), "H2D X");
            else check(cudaMemcpyAsync(dst, X32, sizeof(float) * n, cudaMemcpyHostToDevice, g.copy), "H2D X");
        }
        if (g.needs_labels)
            check(cudaMemcpyAsync(g.lstage[k], labels, sizeof(int) * cfg_.batch, cudaMemcpyHostToDevice, g.copy),
                  "H2D labels");
        check(cudaEventRecord(g.ev_copied[k], g.copy), "record");
    }
}

// Phase 2: staging slot k -> the step's input buffers (padded NHWC / im2col
// rows / padded dense rows of X, the labels) on each GPU's main stream,
// ordered after the previous step (whose first-layer weight gradient reads X).
void Session::convert_staged(int k, bool is64) {
    const int I0 = net_.dims[0];
    const int b = cfg_.batch;
    Gpu& g0 = *gpus_[0];
    for (auto& gp : gpus_) {
        Gpu& g = *gp;
        check(cudaSetDevice(g.ordinal), "cudaSetDevice");
        if (g.ordinal != g0.ordinal) check(cudaStreamWaitEvent(g.main, g0.ev_done, 0), "wait");
        check(cudaStreamWaitEvent(g.main, g.ev_copied[k], 0), "wait");
        const double* x64 = is64 ? (k ? g.xstage2 : g.xstage) : nullptr;
        const float* x32 = is64 ? nullptr : reinterpret_cast<const float*>(k ? g.xstage2 : g.xstage);
        if (g.needs_x && lay_[0].kind == 2) {
            const LayerInfo& c = net_.info[0];
            check(launch_im2col_input(x64, x32, b, c.H, c.W, c.in_units, c.ksz, c.pad, g.act.at(0), lay_[0].ld, g.main),
                  "im2col X");
        } else if (g.needs_x && lay_[0].kind == 0) {
            // conv input: host NHWC rows -> padded NHWC (zero border stays from allocation)
            const LayerInfo& c = net_.info[0];
            check(launch_pad_input(x64, x32, b, c.H, c.W, c.in_units, g.act.at(0), c.pad, lay_[0].ld, g.main), "pad X");
        } else if (g.needs_x) {
            float* x = g.act.at(0);
            if (is64) {
                check(launch_convert_f64(x64, b, I0, x, ld_of(I0), g.main), "convert X");
            } else {
                check(cudaMemcpy2DAsync(x, sizeof(float) * ld_of(I0), x32, sizeof(float) * I0, sizeof(float) * I0, b,
                                        cudaMemcpyDeviceToDevice, g.main), "copy X");
            }
        }
        if (g.needs_labels)
            check(cudaMemcpyAsync(g.labels, g.lstage[k], sizeof(int) * b, cudaMemcpyDeviceToDevice, g.main), "labels");
        check(cudaEventRecord(g.ev_consumed[k], g.main), "record");
        check(cudaEventRecord(g.ev_loaded, g.main), "record");
        if (g.ordinal != g0.ordinal) {
            check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
            check(cudaStreamWaitEvent(g0.main, g.ev_loaded, 0), "wait");
        }
    }
}

void Session::step(int iterations) {
    Gpu& g0 = *gpus_[0];
    for (int it = 0; it < iterations; ++it) {
        if (graph_ok_) {
            check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
            check(cudaGraphLaunch(graph_exec_, g0.main), "graph launch");
        } else {
            enqueue_iteration();
        }
        ++steps_enqueued_;
    }
    check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
    check(cudaEventRecord(g0.ev_done, g0.main), "record");
}

void Session::sync() {
    Gpu& g0 = *gpus_[0];
    check(cudaSetDevice(g0.ordinal), "cudaSetDevice");
    // watchdog in the spirit of the reference's receive deadline (:46-61)
    const auto deadline = std::chrono::steady_clock::now() +
                          std::chrono::duration<double>(cfg_.timeout_s * std::max(1, steps_enqueued_));
    while (true) {
        cudaError_t e = cudaEventQuery(g0.ev_done);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) cuda_fail(e, "step");
        if (std::chrono::steady_clock::now() > deadline)
            throw std::runtime_error("handoff deadlock: timed out waiting for step " + S(steps_enqueued_));
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    int first_bad = 0;
    for (auto& gp : gpus_) {
        check(cudaSetDevice(gp->ordinal), "cudaSetDevice");
        check(cudaDeviceSynchronize(), "step");
        StepState st;
        check(cudaMemcpy(&st, gp->st, sizeof(st), cudaMemcpyDeviceToHost), "D2H state");
        if (st.diverged_first && (first_bad == 0 || st.diverged_first < first_bad)) first_bad = st.diverged_first;
    }
    if (first_bad) throw std::runtime_error("diverged at iteration " + S(first_bad));
    if (pending_acc_error_ && steps_enqueued_ > 0) throw std::invalid_argument("accuracy expects binary labels");
}

void Session::history(double* loss, double* acc, int cap, int* count) {
    sync();
    Gpu& g = gpu_of(main_gpu_);
    const int n = std::min(steps_enqueued_, hist_cap_);
    const int first = steps_enqueued_ - n;
    std::vector<double> lh(hist_cap_), ah(hist_cap_);
    check(cudaSetDevice(g.ordinal), "cudaSetDevice");
    check(cudaMemcpy(lh.data(), g.loss_hist, sizeof(double) * hist_cap_, cudaMemcpyDeviceToHost), "D2H hist");
    check(cudaMemcpy(ah.data(), g.acc_hist, sizeof(double) * hist_cap_, cudaMemcpyDeviceToHost), "D2H hist");
    const int k = std::min(n, cap);
    for (int i = 0; i < k; ++i) {
        if (loss) loss[i] = lh[(first + i) % hist_cap_];
        if (acc) acc[i] = ah[(first + i) % hist_cap_];
    }
    if (count) *count = n;
}

double Session::step_host(const double* X64, const float* X32, const int* labels) {
    load_batch(X64, X32, labels);
    step(1);
    Gpu& g = gpu_of(main_gpu_);
    if (loss_pinned_ == nullptr) check(cudaMallocHost(&loss_pinned_, 2 * sizeof(double)), "pinned loss");
    check(cudaSetDevice(g.ordinal), "cudaSetDevice");
    if (g.ordinal != gpus_[0]->ordinal) check(cudaStreamWaitEvent(g.main, gpus_[0]->ev_done, 0), "wait");
    check(cudaMemcpyAsync(loss_pinned_, g.loss_hist + (steps_enqueued_ - 1) % hist_cap_, sizeof(double),
                          cudaMemcpyDeviceToHost, g.main),
          "D2H loss");
    check(cudaStreamSynchronize(g.main), "sync");
    return *loss_pinned_;
}

// Streaming entry: batch t is staged into slot t % 2 on the copy streams
// while step t - 1 still runs, converted and stepped behind it, and its loss
// read back asynchronously; returns the loss of step t - 1 (NaN on the first
// call of a stream), so at most two steps are in flight and the host -> device
// copy of the next batch overlaps the current step.
double Session::step_host_pipelined(const double* X64, const float* X32, const int* labels) {
    Gpu& g = gpu_of(main_gpu_);
    if (loss_pinned_ == nullptr) check(cudaMallocHost(&loss_pinned_, 2 * sizeof(double)), "pinned loss");
    if (ev_loss_[0] == nullptr) {
        check(cudaSetDevice(g.ordinal), "cudaSetDevice");
        for (auto& e : ev_loss_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    const int k = stream_steps_ & 1;
    stage_batch(X64, X32, labels, k);
    convert_staged(k, X64 != nullptr);
    step(1);
    check(cudaSetDevice(g.ordinal), "cudaSetDevice");
    if (g.ordinal != gpus_[0]->ordinal) check(cudaStreamWaitEvent(g.main, gpus_[0]->ev_done, 0), "wait");
    check(cudaMemcpyAsync(loss_pinned_ + k, g.loss_hist + (steps_enqueued_ - 1) % hist_cap_, sizeof(double),
                          cudaMemcpyDeviceToHost, g.main),
          "D2H loss");
    check(cudaEventRecord(ev_loss_[k], g.main), "record");
    ++stream_steps_;
    if (stream_steps_ == 1) return std::nan("");
    check(cudaEventSynchronize(ev_loss_[k ^ 1]), "loss of the previous step");
    return loss_pinned_[k ^ 1];
}

double Session::last_loss() {
    if (steps_enqueued_ == 0) return 0.0;
    Gpu& g = gpu_of(main_gpu_);
    double v = 0.0;
    check(cudaSetDevice(gpus_[0]->ordinal), "cudaSetDevice");
    check(cudaEventSynchronize(gpus_[0]->ev_done), "sync");
    check(cudaSetDevice(g.ordinal), "cudaSetDevice");
    check(cudaMemcpy(&v, g.loss_hist + (steps_enqueued_ - 1) % hist_cap_, sizeof(double), cudaMemcpyDeviceToHost),
          "D2H loss");
    return v;
}

void Session::get_net(double* W, double* b) {
    sync();
    const int L = net_.L();
    size_t wo = 0, bo = 0;
    std::vector<float> tmp;
    for (int l = 1; l <= L; ++l) {
        const LayerInfo& li = net_.info[l - 1];
        const int hc = li.host_wcols();
        for (int wi : layer_workers_[l]) {
            Worker& w = *workers_[wi];
            WLayer& wl = w.at(l);
            if (!wl.contributor) continue;  // replicated: rank 0 copy (:698)
            tmp.resize(static_cast<size_t>(wl.u) * wl.ldw);
            check(cudaSetDevice(w.gpu), "cudaSetDevice");
            check(cudaMemcpy(tmp.data(), wl.W, sizeof(float) * tmp.size(), cudaMemcpyDeviceToHost), "D2H W");
            for (int r = 0; r < wl.u; ++r) {
                double* dst = W + wo + static_cast<size_t>(wl.lo + r) * hc;
                const float* src = tmp.data() + static_cast<size_t>(r) * wl.ldw;
                if (li.kind == 1 && !li.im2col && !li.generic) {
                    for (int t = 0; t < li.ksz * li.ksz; ++t)
                        for (int c = 0; c < li.in_units; ++c) dst[t * li.in_units + c] = src[t * li.ck() + c];
                } else {
                    for (int c = 0; c < hc; ++c) dst[c] = src[c];
                }
            }
            std::vector<float> bb(wl.u);
            check(cudaMemcpy(bb.data(), wl.bias, sizeof(float) * wl.u, cudaMemcpyDeviceToHost), "D2H b");
            for (int r = 0; r < wl.u; ++r) b[bo + wl.lo + r] = bb[r];
        }
        wo += static_cast<size_t>(hc) * li.out_units;
        bo += li.out_units;
    }
}

size_t Session::read_tensor(int kind, int layer, int device, double* out, size_t cap) {
    sync();
    const int L = net_.L();
    const int b = cfg_.batch;
    if (layer < 1 || layer > L) throw std::out_of_range("layer " + S(layer) + " out of range");
    std::vector<float> tmp;
    auto fetch = [&](const float* p, int ord, int rows, int cols, long long ld) {
        tmp.resize(static_cast<size_t>(rows) * ld);
        check(cudaSetDevice(ord), "cudaSetDevice");
        check(cudaMemcpy(tmp.data(), p, sizeof(float) * tmp.size(), cudaMemcpyDeviceToHost), "D2H tensor");
        const size_t n = static_cast<size_t>(rows) * cols;
        if (out != nullptr) {
            if (cap < n) throw std::length_error("tensor buffer too small");
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < cols; ++c) out[static_cast<size_t>(r) * cols + c] = tmp[static_cast<size_t>(r) * ld + c];
        }
        return n;
    };
    auto raw = [&](const float* p, int ord, size_t nfloats) {
        tmp.resize(nfloats);
        check(cudaSetDevice(ord), "cudaSetDevice");
        check(cudaMemcpy(tmp.data(), p, sizeof(float) * nfloats, cudaMemcpyDeviceToHost), "D2H tensor");
    };
    const int F = net_.dims[layer];
    const bool softmax_head = layer == L && net_.acts[L - 1] == 2;
    if (kind == 0 || kind == 1) {
        if (kind == 1 && !softmax_head) throw std::invalid_argument("pre-activation is kept only for the softmax head");
        if (softmax_head) {
            int ord = workers_[layer_workers_[L].front()]->gpu;
            size_t n = fetch(q_buf(ord), ord, b, F, ld_of(F));
            if (kind == 0 && out != nullptr) {
                for (int r = 0; r < b; ++r) {
                    double* row = out + static_cast<size_t>(r) * F;
                    double mx = row[0];
                    for (int c = 1; c < F; ++c) mx = std::max(mx, row[c]);
                    double s = 0.0;
                    for (int c = 0; c < F; ++c) s += (row[c] = std::exp(row[c] - mx));
                    for (int c = 0; c < F; ++c) row[c] /= s;
                }
            }
            return n;
        }
        const LayerInfo& li = net_.info[layer - 1];
        for (auto& gp : gpus_) {
            auto it = gp->act.find(layer);
            if (it == gp->act.end()) continue;
            if (li.kind == 0) return fetch(it->second, gp->ordinal, b, F, ld_of(F));
            // conv output, returned per sample in (h, w, c) order
            const ActLayout& a = lay_[layer];
            const int Hq = li.Hq(), Wq = li.Wq(), Cc = li.out_units;
            const long long per = img_elems(layer);
            raw(it->second, gp->ordinal, static_cast<size_t>(b) * per);
            const size_t n = static_cast<size_t>(b) * Hq * Wq * Cc;
            if (out != nullptr) {
                if (cap < n) throw std::length_error("tensor buffer too small");
                for (int i = 0; i < b; ++i)
                    for (int y = 0; y < Hq; ++y)
                        for (int x = 0; x < Wq; ++x)
                            for (int c = 0; c < Cc; ++c) {
                                const long long src = a.kind == 0
                                    ? ((static_cast<long long>(i) * a.hp + y + a.pad) * a.wp + x + a.pad) * a.ld + c
                                    : i * a.ld + (static_cast<long long>(c) * Hq + y) * Wq + x;
                                out[((static_cast<size_t>(i) * Hq + y) * Wq + x) * Cc + c] = tmp[src];
                            }
            }
            return n;
        }
        throw std::runtime_error("internal: activation not resident");
    }
    if (kind == 2) {
        const LayerInfo& li = net_.info[layer - 1];
        for (int wi : layer_workers_[layer]) {
            Worker& w = *workers_[wi];
            if (w.device != device) continue;
            WLayer& wl = w.at(layer);
            if (li.kind == 0) return fetch(wl.delta, w.gpu, b, wl.u, wl.ldd);
            const int q = li.dq(), Ho = li.Ho(), Wo = li.Wo();
            const long long per = wl.delta_img;
            raw(wl.delta, w.gpu, static_cast<size_t>(b) * per);
            const size_t n = static_cast<size_t>(b) * Ho * Wo * wl.u;
            if (out != nullptr) {
                if (cap < n) throw std::length_error("tensor buffer too small");
                for (int i = 0; i < b; ++i)
                    for (int y = 0; y < Ho; ++y)
                        for (int x = 0; x < Wo; ++x)
                            for (int c = 0; c < wl.u; ++c)
                                out[((static_cast<size_t>(i) * Ho + y) * Wo + x) * wl.u + c] =
                                    tmp[i * per + ((static_cast<long long>(y + q)) * (Wo + 2 * q) + x + q) * wl.ldd + c];
            }
            return n;
        }
        throw std::out_of_range("device " + S(device) + " holds no shard of layer " + S(layer));
    }
    throw std::invalid_argument("unknown tensor kind " + S(kind));
}

}  // namespace ppb
