// C entry points of the planner (declared in include/pipeplan_b200.h).
#include <cstring>
#include <vector>

#include "capi_common.h"
#include "planner.h"

using namespace ppb;

namespace {

Chain make_chain(const int* fan_in, const int* fan_out, const double* fwd, int L) {
    if (L < 0 || (L > 0 && (fan_in == nullptr || fan_out == nullptr)))
        throw std::invalid_argument("chain: null dimension arrays");
    Chain g;
    g.fan_in.assign(fan_in, fan_in + L);
    g.fan_out.assign(fan_out, fan_out + L);
    if (fwd != nullptr) g.fwd_flops.assign(fwd, fwd + L);
    return g;
}

void emit(const Plan& p, int* out, int cap, int* out_len) {
    const std::vector<int> f = plan_to_flat(p);
    if (out_len) *out_len = static_cast<int>(f.size());
    if (out != nullptr && cap > 0) {
        if (cap < static_cast<int>(f.size())) throw std::length_error("plan buffer too small");
        std::memcpy(out, f.data(), sizeof(int) * f.size());
    }
}

}  // namespace

extern "C" int ppb_split_layer(int layer_id, int fan_out, const int* devices, int n,
                               int replicate_narrow, int* out_lo, int* out_hi, int* out_replicated) {
    return ppb_guard([&] {
        std::vector<int> devs(n > 0 ? n : 0);
        for (int k = 0; k < n; ++k) devs[k] = devices ? devices[k] : k + 1;
        auto shards = split_layer(layer_id, fan_out, devs, replicate_narrow != 0);
        for (size_t k = 0; k < shards.size(); ++k) {
            out_lo[k] = shards[k].lo;
            out_hi[k] = shards[k].hi;
            out_replicated[k] = shards[k].replicated ? 1 : 0;
        }
    });
}

extern "C" int ppb_split_microbatches(int b, int m, int* out_sizes) {
    return ppb_guard([&] {
        auto v = split_microbatches(b, m);
        std::memcpy(out_sizes, v.data(), sizeof(int) * v.size());
    });
}

extern "C" int ppb_build_plan(const int* fan_in, const int* fan_out, const double* fwd_flops, int L,
                              int n, int Z, int replicate_narrow, int* out, int cap, int* out_len) {
    return ppb_guard([&] {
        emit(build_plan(make_chain(fan_in, fan_out, fwd_flops, L), n, Z, replicate_narrow != 0), out,
             cap, out_len);
    });
}

extern "C" int ppb_build_staged_plan(const int* fan_in, const int* fan_out, const double* fwd_flops,
                                     int L, const int* groups, const int* group_sizes, int Z,
                                     int replicate_narrow, int* out, int cap, int* out_len) {
    return ppb_guard([&] {
        std::vector<std::vector<int>> g;
        int off = 0;
        for (int j = 0; j < Z; ++j) {
            g.emplace_back(groups + off, groups + off + group_sizes[j]);
            off += group_sizes[j];
        }
        emit(build_staged_plan(make_chain(fan_in, fan_out, fwd_flops, L), g, replicate_narrow != 0),
             out, cap, out_len);
    });
}

extern "C" int ppb_build_plan_with_cuts(const int* fan_in, const int* fan_out, int L, int n,
                                        const int* cuts, int ncuts, int replicate_narrow, int* out,
                                        int cap, int* out_len) {
    return ppb_guard([&] {
        std::vector<int> c(cuts, cuts + ncuts);
        emit(build_plan_with_cuts(make_chain(fan_in, fan_out, nullptr, L), n, c, replicate_narrow != 0),
             out, cap, out_len);
    });
}

extern "C" int ppb_merge_submodules(int* plan, int plan_len, const int* group, int group_len) {
    return ppb_guard([&] {
        Plan p = merge_submodules(plan_from_flat(plan, plan_len),
                                  std::vector<int>(group, group + group_len));
        emit(p, plan, plan_len, nullptr);
    });
}

extern "C" int ppb_merge_all(int* plan, int plan_len) {
    return ppb_guard([&] { emit(merge_all(plan_from_flat(plan, plan_len)), plan, plan_len, nullptr); });
}

extern "C" int ppb_serialize_plan(const int* plan, int plan_len, const char* provenance, char* out, size_t cap,
                                  size_t* out_len) {
    return ppb_guard([&] {
        std::vector<std::string> prov;
        if (provenance != nullptr && *provenance) {
            std::string s(provenance);
            size_t a = 0;
            while (true) {
                const size_t b = s.find('\n', a);
                prov.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
                if (b == std::string::npos) break;
                a = b + 1;
            }
        }
        const std::string t = serialize_plan(plan_from_flat(plan, plan_len), prov);
        if (out_len) *out_len = t.size();
        if (out != nullptr && cap > 0) {
            if (cap <= t.size()) throw std::length_error("plan text buffer too small");
            std::memcpy(out, t.c_str(), t.size() + 1);
        }
    });
}

extern "C" int ppb_parse_plan(const char* text, int* out, int cap, int* out_len, char* provenance, size_t prov_cap) {
    return ppb_guard([&] {
        if (text == nullptr) throw std::invalid_argument("null plan text");
        std::vector<std::string> prov;
        const Plan p = parse_plan(text, &prov);
        emit(p, out, cap, out_len);
        if (provenance != nullptr && prov_cap > 0) {
            std::string joined;
            for (size_t i = 0; i < prov.size(); ++i) joined += (i ? "\n" : "") + prov[i];
            if (prov_cap <= joined.size()) throw std::length_error("provenance buffer too small");
            std::memcpy(provenance, joined.c_str(), joined.size() + 1);
        }
    });
}

extern "C" int ppb_validate_plan(const int* plan, int plan_len, const int* fan_in,
                                 const int* fan_out, int L, int num_cluster_devices) {
    return ppb_guard([&] {
        validate_plan(plan_from_flat(plan, plan_len), make_chain(fan_in, fan_out, nullptr, L),
                      num_cluster_devices);
    });
}
