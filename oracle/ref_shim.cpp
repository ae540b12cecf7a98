// ref_shim.cpp — extern "C" harness around the UNMODIFIED reference library
// (compiled by oracle/Makefile from /root/reference/proj/src into
// oracle/_ref/).  TEST INFRASTRUCTURE ONLY: used to generate / check golden
// fixtures (tests/golden/make_golden.py), to pin the C restatement
// (oracle/pipeplan_oracle.c), and as bench.py's `--impl reference` arm.
//
// Plans cross this boundary in the flat encoding of include/pipeplan_b200.h;
// exceptions become return codes (1 invalid_argument, 2 runtime_error,
// 3 out_of_range) with the reference's message copied to `err`.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pipeplan/partition.hpp"
#include "pipeplan/schedule.hpp"
#include "pipeplan/tinynet.hpp"
#include "pipeplan/train_partitioned.hpp"
#include "pipeplan/verify.hpp"

using namespace pipeplan;

namespace {

int run(char* err, size_t errlen, const std::function<void()>& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        if (err && errlen) snprintf(err, errlen, "%s", e.what());
        return 1;
    } catch (const std::out_of_range& e) {
        if (err && errlen) snprintf(err, errlen, "%s", e.what());
        return 3;
    } catch (const std::exception& e) {
        if (err && errlen) snprintf(err, errlen, "%s", e.what());
        return 2;
    }
}

TinyNet make_net(const int* dims, const int* acts, int L, const double* W, const double* b) {
    TinyNet net;
    size_t wo = 0, bo = 0;
    for (int l = 0; l < L; ++l) {
        TinyLayer layer;
        layer.weights = Matrix(dims[l + 1], dims[l]);
        std::memcpy(layer.weights.v.data(), W + wo, sizeof(double) * layer.weights.v.size());
        layer.bias.assign(b + bo, b + bo + dims[l + 1]);
        layer.act = static_cast<ActKind>(acts[l]);
        wo += layer.weights.v.size();
        bo += layer.bias.size();
        net.layers.push_back(std::move(layer));
    }
    return net;
}

void dump_net(const TinyNet& net, double* W, double* b) {
    size_t wo = 0, bo = 0;
    for (const TinyLayer& l : net.layers) {
        std::memcpy(W + wo, l.weights.v.data(), sizeof(double) * l.weights.v.size());
        std::memcpy(b + bo, l.bias.data(), sizeof(double) * l.bias.size());
        wo += l.weights.v.size();
        bo += l.bias.size();
    }
}

ModelGraph chain(const int* fan_in, const int* fan_out, int L) {
    ModelGraph g;
    g.name = "chain";
    for (int l = 0; l < L; ++l) {
        LayerSpec s;
        s.id = l + 1;
        s.kind = LayerKind::dense;
        s.fan_in = fan_in[l];
        s.fan_out = fan_out[l];
        g.layers.push_back(s);
    }
    return default_costs(g, 8.0);  // as model_graph_of, tinynet.cpp:463-476
}

std::vector<int> flatten(const PartitionPlan& p) {
    std::vector<int> f{p.n, p.num_submodules()};
    for (const SubModule& sm : p.submodules) {
        f.push_back(sm.index);
        f.push_back(sm.first_layer);
        f.push_back(sm.last_layer);
        f.push_back(static_cast<int>(sm.devices.size()));
        for (int d : sm.devices) f.push_back(d);
        for (const auto& row : sm.shards)
            for (const Shard& s : row) {
                f.push_back(s.layer_id);
                f.push_back(s.device_id);
                f.push_back(s.lo);
                f.push_back(s.hi);
                f.push_back(s.replicated ? 1 : 0);
            }
    }
    for (BoundaryKind k : p.boundaries) f.push_back(k == BoundaryKind::direct ? 1 : 0);
    return f;
}

PartitionPlan unflatten(const int* f, int len) {
    PartitionPlan p;
    int r = 0;
    auto next = [&]() {
        if (r >= len) throw std::runtime_error("malformed plan encoding");
        return f[r++];
    };
    p.n = next();
    const int Z = next();
    for (int j = 0; j < Z; ++j) {
        SubModule sm;
        sm.index = next();
        sm.first_layer = next();
        sm.last_layer = next();
        const int D = next();
        for (int d = 0; d < D; ++d) sm.devices.push_back(next());
        for (int l = sm.first_layer; l <= sm.last_layer; ++l) {
            std::vector<Shard> row;
            for (int d = 0; d < D; ++d) {
                Shard s;
                s.layer_id = next();
                s.device_id = next();
                s.lo = next();
                s.hi = next();
                s.replicated = next() != 0;
                row.push_back(s);
            }
            sm.shards.push_back(row);
        }
        p.submodules.push_back(std::move(sm));
    }
    for (int k = 0; k + 1 < Z; ++k)
        p.boundaries.push_back(next() ? BoundaryKind::direct : BoundaryKind::concat_repartition);
    return p;
}

int emit(const std::vector<int>& f, int* out, int cap, int* out_len) {
    *out_len = static_cast<int>(f.size());
    if (out && cap >= static_cast<int>(f.size())) std::memcpy(out, f.data(), sizeof(int) * f.size());
    return 0;
}

}  // namespace

extern "C" {

void ref_init_net(const int* dims, const int* acts, int L, uint64_t seed, double* W, double* b) {
    std::vector<int> d(dims, dims + L + 1);
    std::vector<ActKind> a;
    for (int l = 0; l < L; ++l) a.push_back(static_cast<ActKind>(acts[l]));
    dump_net(init_net(d, a, seed), W, b);
}

void ref_make_blobs(int samples, int features, double separation, uint64_t seed, double* X,
                    int* labels) {
    Batch bt = make_blobs(samples, features, separation, seed);
    std::memcpy(X, bt.X.v.data(), sizeof(double) * bt.X.v.size());
    std::memcpy(labels, bt.labels.data(), sizeof(int) * bt.labels.size());
}

int ref_split_layer(int layer_id, int fan_out, const int* devices, int n, int replicate, int* lo,
                    int* hi, int* rep, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        LayerSpec s;
        s.id = layer_id;
        s.fan_in = 1;
        s.fan_out = fan_out;
        std::vector<int> devs(devices, devices + n);
        auto shards = split_layer(s, devs, replicate != 0);
        for (size_t k = 0; k < shards.size(); ++k) {
            lo[k] = shards[k].lo;
            hi[k] = shards[k].hi;
            rep[k] = shards[k].replicated ? 1 : 0;
        }
    });
}

int ref_split_microbatches(int b, int m, int* sizes, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        auto v = split_microbatches(b, m);
        std::memcpy(sizes, v.data(), sizeof(int) * v.size());
    });
}

int ref_build_plan(const int* fan_in, const int* fan_out, int L, int n, int Z, int replicate,
                   int* out, int cap, int* out_len, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        emit(flatten(build_plan(chain(fan_in, fan_out, L), n, Z, replicate != 0)), out, cap, out_len);
    });
}

int ref_build_staged_plan(const int* fan_in, const int* fan_out, int L, const int* groups,
                          const int* sizes, int Z, int replicate, int* out, int cap, int* out_len,
                          char* err, size_t errlen) {
    return run(err, errlen, [&] {
        std::vector<std::vector<int>> g;
        int off = 0;
        for (int j = 0; j < Z; ++j) {
            g.emplace_back(groups + off, groups + off + sizes[j]);
            off += sizes[j];
        }
        emit(flatten(build_staged_plan(chain(fan_in, fan_out, L), g, replicate != 0)), out, cap,
             out_len);
    });
}

int ref_build_plan_with_cuts(const int* fan_in, const int* fan_out, int L, int n, const int* cuts,
                             int ncuts, int replicate, int* out, int cap, int* out_len, char* err,
                             size_t errlen) {
    return run(err, errlen, [&] {
        std::vector<int> c(cuts, cuts + ncuts);
        emit(flatten(build_plan_with_cuts(chain(fan_in, fan_out, L), n, c, replicate != 0)), out,
             cap, out_len);
    });
}

int ref_merge_submodules(int* plan, int len, const int* group, int glen, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        PartitionPlan p = merge_submodules(unflatten(plan, len), std::vector<int>(group, group + glen));
        auto f = flatten(p);
        std::memcpy(plan, f.data(), sizeof(int) * f.size());
    });
}

int ref_validate_plan(const int* plan, int len, const int* fan_in, const int* fan_out, int L,
                      char* err, size_t errlen) {
    return run(err, errlen, [&] { validate_plan(unflatten(plan, len), chain(fan_in, fan_out, L)); });
}

int ref_forward(const int* dims, const int* acts, int L, const double* W, const double* b,
                const double* X, int batch, double* acts_out, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        TinyNet net = make_net(dims, acts, L, W, b);
        Matrix x(batch, dims[0]);
        std::memcpy(x.v.data(), X, sizeof(double) * x.v.size());
        ActivationTape tape = forward(net, x);
        size_t off = 0;
        for (int l = 1; l <= L; ++l) {
            std::memcpy(acts_out + off, tape.a[l].v.data(), sizeof(double) * tape.a[l].v.size());
            off += tape.a[l].v.size();
        }
    });
}

static Batch make_batch(const double* X, const int* labels, int batch, int features) {
    Batch bt;
    bt.X = Matrix(batch, features);
    std::memcpy(bt.X.v.data(), X, sizeof(double) * bt.X.v.size());
    bt.labels.assign(labels, labels + batch);
    return bt;
}

int ref_train_sequential(const int* dims, const int* acts, int L, const double* W, const double* b,
                         const double* X, const int* labels, int batch, double alpha0,
                         double decay, int loss, int iterations, double* W_out, double* b_out,
                         double* loss_hist, double* acc_hist, char* err, size_t errlen) {
    return run(err, errlen, [&] {
        TrainConfig cfg;
        cfg.alpha0 = alpha0;
        cfg.decay = decay;
        cfg.loss = static_cast<LossKind>(loss);
        cfg.iterations = iterations;
        TrainResult r = train_sequential(make_net(dims, acts, L, W, b),
                                         make_batch(X, labels, batch, dims[0]), cfg);
        dump_net(r.net, W_out, b_out);
        std::memcpy(loss_hist, r.loss_history.data(), sizeof(double) * r.loss_history.size());
        std::memcpy(acc_hist, r.acc_history.data(), sizeof(double) * r.acc_history.size());
    });
}

int ref_train_partitioned(const int* dims, const int* acts, int L, const double* W,
                          const double* b, const double* X, const int* labels, int batch,
                          const int* plan, int plan_len, int m, int mode, double alpha0,
                          double decay, int loss, int iterations, double timeout_s, double* W_out,
                          double* b_out, double* loss_hist, double* acc_hist, char* err,
                          size_t errlen) {
    return run(err, errlen, [&] {
        TrainConfig cfg;
        cfg.alpha0 = alpha0;
        cfg.decay = decay;
        cfg.loss = static_cast<LossKind>(loss);
        cfg.iterations = iterations;
        PartitionedTrainOptions opts;
        opts.receive_timeout_s = timeout_s;
        TrainResult r = train_partitioned(make_net(dims, acts, L, W, b),
                                          make_batch(X, labels, batch, dims[0]), cfg,
                                          unflatten(plan, plan_len), m,
                                          static_cast<UpdateMode>(mode), opts);
        dump_net(r.net, W_out, b_out);
        std::memcpy(loss_hist, r.loss_history.data(), sizeof(double) * r.loss_history.size());
        std::memcpy(acc_hist, r.acc_history.data(), sizeof(double) * r.acc_history.size());
    });
}

// serialize_plan (src/partition.cpp:303-331); provenance = '\n'-joined entries.
int ref_serialize_plan(const int* plan, int len, const char* provenance, char* out, size_t cap, size_t* out_len,
                       char* err, size_t errlen) {
    return run(err, errlen, [&] {
        PartitionPlan p = unflatten(plan, len);
        if (provenance && *provenance) {
            std::string s(provenance), item;
            size_t a = 0;
            while (true) {
                size_t b = s.find('\n', a);
                p.provenance.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
                if (b == std::string::npos) break;
                a = b + 1;
            }
        }
        const std::string t = serialize_plan(p);
        *out_len = t.size();
        if (out && cap > t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
    });
}

// parse_plan (src/partition.cpp:333-384) -> flat plan.
int ref_parse_plan(const char* text, int* out, int cap, int* out_len, char* err, size_t errlen) {
    return run(err, errlen, [&] { emit(flatten(parse_plan(text)), out, cap, out_len); });
}

// run_verification (src/verify.cpp:104-247): 1 if every property passed.
int ref_run_verification(int seeds, char* report, size_t len) {
    VerifyOptions o;
    o.seeds = seeds;
    VerifyReport r = run_verification(o);
    if (report && len) snprintf(report, len, "%s", verify_report_text(r).c_str());
    return r.all_pass() ? 1 : 0;
}

// draw_instance (src/verify.cpp:20-62) exported flat: the reference's own
// randomized verification instances, so the GPU path can be run on exactly
// the cases run_verification checks.  Buffers: dims[9], acts[8], plan[4096],
// W[4096], b[64], X[256], labels[64].
void ref_draw_instance(uint64_t seed, int* L, int* dims, int* acts, int* n, int* m, int* batch,
                       int* loss, double* alpha0, double* decay, int* iterations, int* plan,
                       int* plan_len, double* W, double* b, double* X, int* labels) {
    VerifyInstance inst = draw_instance(seed);
    *L = inst.net.num_layers();
    dims[0] = inst.net.input_dim();
    for (int l = 0; l < *L; ++l) {
        dims[l + 1] = inst.net.layers[l].fan_out();
        acts[l] = static_cast<int>(inst.net.layers[l].act);
    }
    *n = inst.n;
    *m = inst.m;
    *batch = inst.batch.size();
    *loss = static_cast<int>(inst.cfg.loss);
    *alpha0 = inst.cfg.alpha0;
    *decay = inst.cfg.decay;
    *iterations = inst.cfg.iterations;
    auto f = flatten(inst.plan);
    *plan_len = static_cast<int>(f.size());
    std::memcpy(plan, f.data(), sizeof(int) * f.size());
    dump_net(inst.net, W, b);
    std::memcpy(X, inst.batch.X.v.data(), sizeof(double) * inst.batch.X.v.size());
    std::memcpy(labels, inst.batch.labels.data(), sizeof(int) * inst.batch.labels.size());
}

}  // extern "C"
