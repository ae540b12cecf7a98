// Integer partition planner: the reference's PartitionPlan vocabulary
// (include/pipeplan/partition.hpp:14-47) and the functions the partitioned
// step consumes.  Host-only; results must be bit-exact with the reference
// (tests/test_planner.py checks them against the oracle and the golden
// fixtures generated from the compiled reference).
#pragma once

#include <string>
#include <vector>

namespace ppb {

struct Shard {
    int layer_id = 0;
    int device_id = 0;
    int lo = 0;
    int hi = 0;
    bool replicated = false;
    int units() const { return hi - lo; }
};

struct SubModule {
    int index = 0;
    int first_layer = 0;
    int last_layer = 0;
    std::vector<int> devices;
    std::vector<std::vector<Shard>> shards;  // [layer - first_layer][rank]
    const std::vector<Shard>& layer_shards(int layer) const { return shards.at(layer - first_layer); }
};

enum Boundary : int { kConcat = 0, kDirect = 1 };

struct Plan {
    int n = 0;
    std::vector<SubModule> subs;
    std::vector<int> boundaries;  // Z-1 entries
    int Z() const { return static_cast<int>(subs.size()); }
};

// A dense chain: fan_in[l], fan_out[l] and optional per-layer fwd_flops
// (0 -> default_costs, src/model.cpp:124-137).
struct Chain {
    std::vector<int> fan_in, fan_out;
    std::vector<double> fwd_flops;
    int L() const { return static_cast<int>(fan_out.size()); }
};

std::vector<Shard> split_layer(int layer_id, int fan_out, const std::vector<int>& devices,
                               bool replicate_narrow);
std::vector<int> split_microbatches(int b, int m);
Plan build_plan(const Chain& g, int n, int Z, bool replicate_narrow);
Plan build_staged_plan(const Chain& g, const std::vector<std::vector<int>>& groups,
                       bool replicate_narrow);
Plan build_plan_with_cuts(const Chain& g, int n, const std::vector<int>& cuts,
                          bool replicate_narrow);
Plan merge_submodules(const Plan& p, const std::vector<int>& group);
Plan merge_all(const Plan& p);
void validate_chain(const Chain& g);
void validate_plan(const Plan& p, const Chain& g, int cluster_devices);

// Plan documents (src/partition.cpp:303-384): the reference's JSON schema,
// serialised byte-for-byte like its nlohmann::json dump(2).
std::string serialize_plan(const Plan& p, const std::vector<std::string>& provenance);
Plan parse_plan(const std::string& text, std::vector<std::string>* provenance);

Plan plan_from_flat(const int* flat, int len);
std::vector<int> plan_to_flat(const Plan& p);

}  // namespace ppb
