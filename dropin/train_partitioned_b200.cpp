// Drop-in replacement for the reference's src/train_partitioned.cpp.
//
// A maintainer swaps this file for proj/src/train_partitioned.cpp in the
// pipeplan_core target and links libpipeplan_b200.so:
// every caller of pipeplan::train_partitioned — run_verification
// (src/verify.cpp:122-125), the CLI's verify/demo — then trains on B200s
// through the C ABI (include/pipeplan_b200.h).  Signature, argument meaning
// and exception types/messages are the reference's
// (include/pipeplan/train_partitioned.hpp:24-26).
//
// Environment (optional):
//   PPB_PRECISION = tf32 (default) | fp32
//   PPB_DEVICES   = comma-separated CUDA ordinals for plan devices 1..n
//                   (default: every plan device on cuda:0)
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pipeplan_b200.h"
#include "pipeplan/train_partitioned.hpp"

namespace pipeplan {

namespace {

[[noreturn]] void rethrow(int code) {
    const std::string msg = ppb_last_error();
    if (code == PPB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (code == PPB_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
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

TrainResult train_partitioned(const TinyNet& net, const Batch& batch, const TrainConfig& cfg,
                              const PartitionPlan& plan, int m, UpdateMode mode,
                              const PartitionedTrainOptions& opts) {
    validate_net(net);  // the reference's own entry checks (train_partitioned.cpp:124)
    if (batch.size() != static_cast<int>(batch.labels.size()))
        throw std::invalid_argument("batch rows and label count disagree");
    // the ABI takes a bare pointer to rows x input_dim doubles: a narrower X
    // would be read past its end (the reference throws in matmul_nt,
    // tinynet.cpp:25, called from the shard forward)
    if (batch.X.cols != net.input_dim()) throw std::invalid_argument("matmul_nt: inner dimensions disagree");
    std::vector<int> dims{net.input_dim()}, acts;
    std::vector<double> W, b;
    for (const TinyLayer& l : net.layers) {
        dims.push_back(l.fan_out());
        acts.push_back(static_cast<int>(l.act));
        W.insert(W.end(), l.weights.v.begin(), l.weights.v.end());
        b.insert(b.end(), l.bias.begin(), l.bias.end());
    }
    const std::vector<int> fp = flat_plan(plan);
    int ndev = plan.n;
    for (const SubModule& sm : plan.submodules)
        for (int d : sm.devices) ndev = d > ndev ? d : ndev;
    // default: plan device k+1 on CUDA ordinal k, one plan device per visible
    // GPU (round-robin when the plan has more devices than the box has GPUs);
    // PPB_DEVICES=o1,o2,... overrides
    int ngpu = 0;
    if (ppb_device_count(&ngpu) != PPB_OK || ngpu < 1) ngpu = 1;
    std::vector<int> map(ndev > 0 ? ndev : 1, 0);
    for (size_t k = 0; k < map.size(); ++k) map[k] = static_cast<int>(k % static_cast<size_t>(ngpu));
    if (const char* env = std::getenv("PPB_DEVICES")) {
        std::stringstream ss(env);
        std::string tok;
        for (size_t k = 0; std::getline(ss, tok, ',') && k < map.size(); ++k) map[k] = std::atoi(tok.c_str());
    }
    ppb_context* ctx = nullptr;
    int rc = ppb_context_create(map.data(), static_cast<int>(map.size()), &ctx);
    if (rc != PPB_OK) rethrow(rc);
    ppb_train_config c{cfg.alpha0, cfg.decay, static_cast<int>(cfg.loss), cfg.iterations, cfg.seed};
    ppb_options o;
    ppb_default_options(&o);
    o.receive_timeout_s = opts.receive_timeout_s;
    if (const char* p = std::getenv("PPB_PRECISION")) o.precision = std::strcmp(p, "fp32") == 0 ? PPB_PRECISION_FP32 : PPB_PRECISION_TF32;
    TrainResult r;
    r.net = net;
    std::vector<double> Wo(W.size()), bo(b.size());
    r.loss_history.assign(cfg.iterations, 0.0);
    r.acc_history.assign(cfg.iterations, 0.0);
    rc = ppb_train_partitioned(ctx, dims.data(), acts.data(), static_cast<int>(acts.size()), W.data(), b.data(),
                               batch.X.v.data(), batch.labels.data(), batch.size(), fp.data(),
                               static_cast<int>(fp.size()), m, static_cast<int>(mode), &c, &o, Wo.data(), bo.data(),
                               r.loss_history.data(), r.acc_history.data());
    ppb_context_destroy(ctx);
    if (rc != PPB_OK) rethrow(rc);
    size_t wo = 0, bofs = 0;
    for (TinyLayer& l : r.net.layers) {
        std::memcpy(l.weights.v.data(), Wo.data() + wo, sizeof(double) * l.weights.v.size());
        std::memcpy(l.bias.data(), bo.data() + bofs, sizeof(double) * l.bias.size());
        wo += l.weights.v.size();
        bofs += l.bias.size();
    }
    return r;
}

}  // namespace pipeplan
