// C entry points of the partitioned training step (include/pipeplan_b200.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <vector>

#include "capi_common.h"
#include "planner.h"
#include "session.h"

using namespace ppb;

struct ppb_context {
    std::vector<int> device_map;
};

struct ppb_session {
    std::unique_ptr<Session> s;
};

namespace {

NetDesc make_net(const int* dims, const int* acts, int L) {
    if (L < 1 || dims == nullptr || acts == nullptr) throw std::invalid_argument("net must have at least one layer");
    NetDesc n;
    n.dims.assign(dims, dims + L + 1);
    n.acts.assign(acts, acts + L);
    for (int a : n.acts)
        if (a < 0 || a > 2) throw std::invalid_argument("unknown activation kind " + std::to_string(a));
    return n;
}

SessionConfig make_cfg(int batch, int m, int mode, const ppb_train_config* cfg, const ppb_options* opts) {
    SessionConfig c;
    ppb_train_config dc;
    ppb_default_config(&dc);
    ppb_options dopt;
    ppb_default_options(&dopt);
    if (cfg == nullptr) cfg = &dc;
    if (opts == nullptr) opts = &dopt;
    c.alpha0 = cfg->alpha0;
    c.decay = cfg->decay;
    c.loss = cfg->loss;
    c.batch = batch;
    c.m = m;
    c.mode = mode;
    c.timeout_s = opts->receive_timeout_s > 0 ? opts->receive_timeout_s : 30.0;
    c.precision = opts->precision;
    c.multiclass = opts->multiclass_accuracy;
    c.use_graph = opts->use_graph;
    c.gate = opts->pipeline_gate;
    c.stash = opts->memory_mode;
    c.merge = opts->merge_backend;
    if (c.merge != PPB_MERGE_P2P && c.merge != PPB_MERGE_NCCL) throw std::invalid_argument("unknown merge backend");
    if (c.stash != PPB_MEMORY_STASH_ALL && c.stash != PPB_MEMORY_PROPOSED)
        throw std::invalid_argument("unknown memory mode");
    if (c.loss != 0 && c.loss != 1) throw std::invalid_argument("unknown loss kind");
    if (c.precision != 0 && c.precision != 1) throw std::invalid_argument("unknown precision");
    return c;
}

}  // namespace

extern "C" int ppb_context_create(const int* device_map, int n_logical, ppb_context** out) {
    return ppb_guard([&] {
        if (out == nullptr) throw std::invalid_argument("null output handle");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            throw std::runtime_error("no CUDA device available for pipeplan_b200");
        }
        auto ctx = std::make_unique<ppb_context>();
        for (int k = 0; k < n_logical; ++k) {
            const int ord = device_map ? device_map[k] : k % ndev;
            if (ord < 0 || ord >= ndev)
                throw std::invalid_argument("device map entry " + std::to_string(ord) + " is not a CUDA device");
            ctx->device_map.push_back(ord);
        }
        *out = ctx.release();
    });
}

extern "C" void ppb_context_destroy(ppb_context* ctx) { delete ctx; }

extern "C" int ppb_session_create(ppb_context* ctx, const int* dims, const int* acts, int L,
                                  const double* W, const double* b, int batch, const int* plan,
                                  int plan_len, int m, int mode, const ppb_train_config* cfg,
                                  const ppb_options* opts, ppb_session** out) {
    return ppb_guard([&] {
        if (ctx == nullptr || out == nullptr) throw std::invalid_argument("null context or output handle");
        NetDesc net = make_net(dims, acts, L);
        Plan p;
        try {
            p = plan_from_flat(plan, plan_len);
        } catch (const std::exception& e) {
            throw std::runtime_error(std::string("plan/net shape mismatch: ") + e.what());
        }
        auto s = std::make_unique<ppb_session>();
        s->s = std::make_unique<Session>(ctx->device_map, net, W, b, p, make_cfg(batch, m, mode, cfg, opts));
        *out = s.release();
    });
}

extern "C" void ppb_session_destroy(ppb_session* s) { delete s; }

extern "C" int ppb_session_create_layers(ppb_context* ctx, const ppb_layer* layers, int L, const double* W,
                                         const double* b, int batch, const int* plan, int plan_len, int m,
                                         int mode, const ppb_train_config* cfg, const ppb_options* opts,
                                         ppb_session** out) {
    return ppb_guard([&] {
        if (ctx == nullptr || out == nullptr || layers == nullptr || L < 1)
            throw std::invalid_argument("net must have at least one layer");
        NetDesc net;
        for (int l = 0; l < L; ++l) {
            const ppb_layer& p = layers[l];
            if (p.kind != PPB_LAYER_DENSE && p.kind != PPB_LAYER_CONV)
                throw std::invalid_argument("unknown layer kind " + std::to_string(p.kind));
            if (p.act < 0 || p.act > 2) throw std::invalid_argument("unknown activation kind " + std::to_string(p.act));
            LayerInfo li;
            li.kind = p.kind;
            li.in_units = p.in_units;
            li.out_units = p.out_units;
            li.act = p.act;
            if (p.kind == PPB_LAYER_CONV) {
                li.H = p.height;
                li.W = p.width;
                li.ksz = p.ksize;
                li.pad = p.pad;
                li.pool = p.pool < 1 ? 1 : p.pool;
                li.res_from = p.res_from;
                li.stride = p.stride < 1 ? 1 : p.stride;
                li.pool_avg = p.pool_kind == PPB_POOL_AVG ? 1 : 0;
                if (p.pool_kind != PPB_POOL_MAX && p.pool_kind != PPB_POOL_AVG)
                    throw std::invalid_argument("unknown pool kind " + std::to_string(p.pool_kind));
            }
            net.info.push_back(li);
            net.acts.push_back(p.act);
        }
        net.dims.assign(L + 1, 0);
        Plan pl;
        try {
            pl = plan_from_flat(plan, plan_len);
        } catch (const std::exception& e) {
            throw std::runtime_error(std::string("plan/net shape mismatch: ") + e.what());
        }
        auto s = std::make_unique<ppb_session>();
        s->s = std::make_unique<Session>(ctx->device_map, net, W, b, pl, make_cfg(batch, m, mode, cfg, opts));
        *out = s.release();
    });
}

extern "C" int ppb_train_partitioned_layers(ppb_context* ctx, const ppb_layer* layers, int L, const double* W,
                                            const double* b, const double* X, const int* labels, int batch,
                                            const int* plan, int plan_len, int m, int mode,
                                            const ppb_train_config* cfg, const ppb_options* opts, double* W_out,
                                            double* b_out, double* loss_hist, double* acc_hist) {
    ppb_session* s = nullptr;
    int rc = ppb_session_create_layers(ctx, layers, L, W, b, batch, plan, plan_len, m, mode, cfg, opts, &s);
    if (rc != PPB_OK) return rc;
    std::unique_ptr<ppb_session> guard(s);
    return ppb_guard([&] {
        ppb_train_config dc;
        ppb_default_config(&dc);
        const int iters = cfg ? cfg->iterations : dc.iterations;
        s->s->load_batch(X, nullptr, labels);
        s->s->step(iters);
        s->s->sync();
        int count = 0;
        s->s->history(loss_hist, acc_hist, iters, &count);
        s->s->get_net(W_out, b_out);
    });
}

extern "C" int ppb_session_load_batch(ppb_session* s, const double* X, const int* labels) {
    return ppb_guard([&] { s->s->load_batch(X, nullptr, labels); });
}

extern "C" int ppb_session_load_batch_f32(ppb_session* s, const float* X, const int* labels) {
    return ppb_guard([&] { s->s->load_batch(nullptr, X, labels); });
}

extern "C" int ppb_session_step(ppb_session* s, int iterations) {
    return ppb_guard([&] { s->s->step(iterations); });
}

extern "C" int ppb_session_step_host(ppb_session* s, const float* X, const int* labels, double* loss_out) {
    return ppb_guard([&] {
        const double v = s->s->step_host(nullptr, X, labels);
        if (loss_out) *loss_out = v;
    });
}

extern "C" int ppb_session_step_host_f64(ppb_session* s, const double* X, const int* labels, double* loss_out) {
    return ppb_guard([&] {
        const double v = s->s->step_host(X, nullptr, labels);
        if (loss_out) *loss_out = v;
    });
}

extern "C" int ppb_session_step_host_pipelined(ppb_session* s, const float* X, const double* X64, const int* labels,
                                               double* prev_loss_out) {
    return ppb_guard([&] {
        const double v = s->s->step_host_pipelined(X64, X64 ? nullptr : X, labels);
        if (prev_loss_out) *prev_loss_out = v;
    });
}

extern "C" int ppb_session_sync(ppb_session* s) {
    return ppb_guard([&] { s->s->sync(); });
}

extern "C" int ppb_session_history(ppb_session* s, double* loss_hist, double* acc_hist, int cap, int* count) {
    return ppb_guard([&] { s->s->history(loss_hist, acc_hist, cap, count); });
}

extern "C" int ppb_session_memory(ppb_session* s, size_t* total_bytes, size_t* stash_bytes) {
    return ppb_guard([&] {
        if (total_bytes) *total_bytes = s->s->device_bytes();
        if (stash_bytes) *stash_bytes = s->s->stash_bytes();
    });
}

extern "C" int ppb_session_get_net(ppb_session* s, double* W_out, double* b_out) {
    return ppb_guard([&] { s->s->get_net(W_out, b_out); });
}

extern "C" int ppb_session_read_tensor(ppb_session* s, int kind, int layer, int device, double* out,
                                       size_t cap_elems, size_t* out_elems) {
    return ppb_guard([&] {
        const size_t n = s->s->read_tensor(kind, layer, device, out, cap_elems);
        if (out_elems) *out_elems = n;
    });
}

extern "C" int ppb_session_time_steps(ppb_session* s, int iterations, float* ms_out) {
    return ppb_guard([&] { *ms_out = s->s->time_steps(iterations); });
}

extern "C" int ppb_session_profile(ppb_session* s, int iterations, double* ms, int* count, double* flops,
                                   int nkinds) {
    return ppb_guard([&] { s->s->profile(iterations, ms, count, flops, nkinds); });
}

extern "C" int ppb_session_profile_starts(ppb_session* s, double* start_ms, int* stream_id, int cap, int* count) {
    return ppb_guard([&] { *count = s->s->profile_starts(start_ms, stream_id, cap); });
}

extern "C" int ppb_session_profile_concurrent(ppb_session* s, int iterations) {
    return ppb_guard([&] {
        constexpr int kKinds = OP_NKINDS;
        double ms[kKinds], fl[kKinds];
        int cnt[kKinds];
        s->s->set_profile_serialised(false);
        try {
            s->s->profile(iterations, ms, cnt, fl, kKinds);
        } catch (...) {
            s->s->set_profile_serialised(true);
            throw;
        }
        s->s->set_profile_serialised(true);
    });
}

extern "C" int ppb_session_op_meta(ppb_session* s, int* microbatch, int* device, int* role, int cap, int* count) {
    return ppb_guard([&] { *count = s->s->op_meta(microbatch, device, role, cap); });
}

extern "C" int ppb_session_profile_ops(ppb_session* s, int* kind, int* layer, int* info, double* ms, double* flops,
                                       int cap, int* count) {
    return ppb_guard([&] { *count = s->s->profile_ops(kind, layer, info, ms, flops, cap); });
}

extern "C" int ppb_session_kernels_per_step(ppb_session* s, int* out) {
    return ppb_guard([&] { *out = s->s->kernels_per_step(); });
}

extern "C" int ppb_train_partitioned(ppb_context* ctx, const int* dims, const int* acts, int L,
                                     const double* W, const double* b, const double* X,
                                     const int* labels, int batch, const int* plan, int plan_len,
                                     int m, int mode, const ppb_train_config* cfg,
                                     const ppb_options* opts, double* W_out, double* b_out,
                                     double* loss_hist, double* acc_hist) {
    ppb_session* s = nullptr;
    int rc = ppb_session_create(ctx, dims, acts, L, W, b, batch, plan, plan_len, m, mode, cfg, opts, &s);
    if (rc != PPB_OK) return rc;
    std::unique_ptr<ppb_session> guard(s);
    return ppb_guard([&] {
        ppb_train_config dc;
        ppb_default_config(&dc);
        const int iters = cfg ? cfg->iterations : dc.iterations;
        s->s->load_batch(X, nullptr, labels);
        s->s->step(iters);
        s->s->sync();
        int count = 0;
        s->s->history(loss_hist, acc_hist, iters, &count);
        s->s->get_net(W_out, b_out);
    });
}
