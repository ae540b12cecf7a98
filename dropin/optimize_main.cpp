// Plan selection priced with measured B200 costs.
//
// The reference's cost model (src/cost.cpp:25-69, 151-238) prices a sub-module
// pass as per-sample layer flops / device flops_per_sec.  Here the per-layer
// forward and backward seconds of the partitioned step are MEASURED on the
// B200 (ppb_session_profile / ppb_session_profile_ops on a one-device plan,
// CUDA events around every op, serialised), converted into per-sample
// "effective flops" at a nominal device rate R, and handed to the reference's
// own task_costs / optimize_plan, so the optimiser ranks candidate plans by
// B200 time.  The link is NVLink 5's nominal alpha-beta (2 us, 900 GB/s):
// one GPU is available in this environment, so it is not measured.
//
//   optimize_b200 <dims,comma,separated> <n> [m] [batch] [model_out.json] [cluster_out.json]
//
// Prints the optimiser report for the calibrated model and, for comparison,
// the objective of the default all-layers-over-n plan (build_plan Z=1).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "pipeplan/cost.hpp"
#include "pipeplan/model.hpp"
#include "pipeplan/partition.hpp"
#include "pipeplan/tinynet.hpp"
#include "pipeplan_b200.h"

using namespace pipeplan;

namespace {

void check(int rc, const char* what) {
    if (rc != PPB_OK) {
        std::fprintf(stderr, "%s: %s\n", what, ppb_last_error());
        std::exit(2);
    }
}

std::vector<int> flat_plan(const PartitionPlan& p) {
    std::vector<int> f{p.n, p.num_submodules()};
    for (const SubModule& sm : p.submodules) {
        f.insert(f.end(), {sm.index, sm.first_layer, sm.last_layer, static_cast<int>(sm.devices.size())});
        f.insert(f.end(), sm.devices.begin(), sm.devices.end());
        for (const auto& row : sm.shards)
            for (const Shard& s : row) f.insert(f.end(), {s.layer_id, s.device_id, s.lo, s.hi, s.replicated ? 1 : 0});
    }
    for (BoundaryKind k : p.boundaries) f.push_back(k == BoundaryKind::direct ? PPB_BOUNDARY_DIRECT : PPB_BOUNDARY_CONCAT);
    return f;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <dims> <n> [m] [batch] [model_out] [cluster_out]\n", argv[0]);
        return 2;
    }
    std::vector<int> dims;
    {
        std::stringstream ss(argv[1]);
        std::string t;
        while (std::getline(ss, t, ',')) dims.push_back(std::atoi(t.c_str()));
    }
    const int n = std::atoi(argv[2]);
    const int m = argc > 3 ? std::atoi(argv[3]) : 1;
    const int batch = argc > 4 ? std::atoi(argv[4]) : 512;
    const int L = static_cast<int>(dims.size()) - 1;
    std::vector<ActKind> acts(L, ActKind::relu);
    acts.back() = ActKind::softmax_last;
    const TinyNet net = init_net(dims, acts, 1);

    // ---- measure per-layer fwd / bwd seconds on the B200 (one device, n = 1)
    std::vector<int> d(dims), a;
    std::vector<double> W, b;
    for (const TinyLayer& l : net.layers) {
        a.push_back(static_cast<int>(l.act));
        W.insert(W.end(), l.weights.v.begin(), l.weights.v.end());
        b.insert(b.end(), l.bias.begin(), l.bias.end());
    }
    const PartitionPlan one = build_plan(model_graph_of(net), 1, 1);
    const std::vector<int> fp = flat_plan(one);
    int dev0 = 0;
    ppb_context* ctx = nullptr;
    check(ppb_context_create(&dev0, 1, &ctx), "context");
    ppb_train_config cfg;
    ppb_default_config(&cfg);
    ppb_options opt;
    ppb_default_options(&opt);
    opt.multiclass_accuracy = 1;
    ppb_session* s = nullptr;
    check(ppb_session_create(ctx, d.data(), a.data(), L, W.data(), b.data(), batch, fp.data(),
                             static_cast<int>(fp.size()), 1, 1, &cfg, &opt, &s),
          "session");
    std::vector<float> X(static_cast<size_t>(batch) * dims[0]);
    std::vector<int> y(batch);
    for (size_t i = 0; i < X.size(); ++i) X[i] = static_cast<float>((i * 2654435761u % 1000) / 1000.0 - 0.5);
    for (int i = 0; i < batch; ++i) y[i] = i % dims.back();
    check(ppb_session_load_batch_f32(s, X.data(), y.data()), "load");
    check(ppb_session_step(s, 3), "warm-up");
    check(ppb_session_sync(s), "sync");
    constexpr int kKinds = 11;
    double ms[kKinds], fl[kKinds];
    int cnt[kKinds];
    check(ppb_session_profile(s, 3, ms, cnt, fl, kKinds), "profile");
    int nops = 0;
    check(ppb_session_profile_ops(s, nullptr, nullptr, nullptr, nullptr, nullptr, 0, &nops), "ops");
    std::vector<int> kind(nops), layer(nops), info(nops);
    std::vector<double> oms(nops), ofl(nops);
    check(ppb_session_profile_ops(s, kind.data(), layer.data(), info.data(), oms.data(), ofl.data(), nops, &nops),
          "ops");
    // op kinds (session.h OpKind): 1 fwd GEMM, 4 loss, 9 pool -> forward;
    // 2 dgrad, 3 wgrad, 5 reduce, 6 bias, 10 merge -> backward; ms summed over 3 steps
    std::map<int, double> tf, tb;
    for (int i = 0; i < nops; ++i) {
        const int k = kind[i], l = layer[i];
        if (l < 1 || l > L) continue;
        if (k == 1 || k == 4 || k == 9) tf[l] += oms[i] / 3.0 * 1e-3;
        else if (k == 2 || k == 3 || k == 5 || k == 6 || k == 10) tb[l] += oms[i] / 3.0 * 1e-3;
    }
    ppb_session_destroy(s);
    ppb_context_destroy(ctx);

    // ---- calibrated model: per-sample effective flops at the nominal rate R
    const double R = 806e12;  // TF32 dense peak (the roofline denominator)
    ModelGraph g = model_graph_of(net, "b200-calibrated");
    for (LayerSpec& ls : g.layers) {
        ls.fwd_flops = tf[ls.id] * R / batch;
        ls.bwd_flops = tb[ls.id] * R / batch;
    }
    const ClusterSpec cluster = uniform_cluster(n, R, 180e9, 2e-6, 900e9);
    OptimizeOptions oo;
    oo.m = m;
    oo.microbatch_samples = batch / m;
    oo.replicate_narrow = true;
    const OptimizeResult r = optimize_plan(g, cluster, n, oo);
    CostParams cp;
    cp.cluster = cluster;
    cp.microbatch_samples = batch / m;
    cp.microbatches = m;
    const PartitionPlan base = build_plan(g, n, 1, true);
    const double base_obj = total_cost(task_costs(base, g, cp));
    std::printf("%s\n", serialize_optimizer_report(r).c_str());
    std::printf("{\"baseline_build_plan_Z1_objective_s\": %.9g, \"optimized_objective_s\": %.9g, "
                "\"measured_step_fwd_s\": %.9g, \"measured_step_bwd_s\": %.9g}\n",
                base_obj, r.objective, [&] { double t = 0; for (auto& kv : tf) t += kv.second; return t; }(),
                [&] { double t = 0; for (auto& kv : tb) t += kv.second; return t; }());
    if (argc > 5) std::ofstream(argv[5]) << serialize_model(g);
    if (argc > 6) std::ofstream(argv[6]) << serialize_cluster(cluster);
    return 0;
}
