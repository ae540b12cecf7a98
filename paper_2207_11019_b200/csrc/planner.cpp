// Integer partition planner (host).  Semantics follow the reference planner
// line by line where it matters for bit-exactness:
//   split_layer         src/partition.cpp:15-48   largest remainder, larger shards first
//   balanced_spans      src/partition.cpp:55-82   cut i = argmin |prefix - total*i/Z|, strict <
//   plan_from_spans     src/partition.cpp:84-106  every layer split over the group, boundaries concat
//   build_plan / build_staged_plan / build_plan_with_cuts   :110-155
//   merge_submodules / merge_all                  :157-182
//   validate_plan                                 :232-294
//   split_microbatches  src/schedule.cpp:46-55
#include "planner.h"

#include <cmath>
#include <stdexcept>

namespace ppb {

namespace {

std::string S(long long v) { return std::to_string(v); }

double fwd_cost(const Chain& g, int l /*0-based*/) {
    if (l < static_cast<int>(g.fwd_flops.size()) && g.fwd_flops[l] != 0) return g.fwd_flops[l];
    const double io = static_cast<double>(g.fan_in[l]) * g.fan_out[l];
    return 2.0 * io;
}

std::vector<int> spans(const Chain& g, int Z) {
    const int L = g.L();
    std::vector<double> prefix(L + 1, 0.0);
    for (int l = 1; l <= L; ++l) prefix[l] = prefix[l - 1] + fwd_cost(g, l - 1);
    const double total = prefix[L];
    std::vector<int> cuts;
    int prev = 0;
    for (int i = 1; i < Z; ++i) {
        const double target = total * i / Z;
        const int first = prev + 1, last = L - (Z - i);
        int best = first;
        double best_err = std::abs(prefix[first] - target);
        for (int pos = first + 1; pos <= last; ++pos) {
            const double e = std::abs(prefix[pos] - target);
            if (e < best_err) {
                best_err = e;
                best = pos;
            }
        }
        cuts.push_back(best);
        prev = best;
    }
    return cuts;
}

Plan from_spans(const Chain& g, const std::vector<int>& cuts,
                const std::vector<std::vector<int>>& groups, int n, bool replicate) {
    Plan p;
    p.n = n;
    const int Z = static_cast<int>(groups.size());
    int first = 1;
    for (int j = 0; j < Z; ++j) {
        SubModule sm;
        sm.index = j + 1;
        sm.first_layer = first;
        sm.last_layer = j + 1 < Z ? cuts[j] : g.L();
        sm.devices = groups[j];
        for (int l = sm.first_layer; l <= sm.last_layer; ++l)
            sm.shards.push_back(split_layer(l, g.fan_out[l - 1], sm.devices, replicate));
        first = sm.last_layer + 1;
        p.subs.push_back(std::move(sm));
    }
    p.boundaries.assign(Z - 1, kConcat);
    return p;
}

std::vector<int> iota1(int n) {
    std::vector<int> v(n);
    for (int i = 0; i < n; ++i) v[i] = i + 1;
    return v;
}

void check_z(const Chain& g, int Z) {
    if (Z < 1 || Z > g.L())
        throw std::runtime_error("Z exceeds layer count (Z=" + S(Z) + ", L=" + S(g.L()) + ")");
}

}  // namespace

std::vector<Shard> split_layer(int layer_id, int fan_out, const std::vector<int>& devices,
                               bool replicate_narrow) {
    const int n = static_cast<int>(devices.size());
    if (n < 1) throw std::invalid_argument("split_layer: need at least one device");
    std::vector<Shard> out(n);
    if (fan_out < n) {
        if (!replicate_narrow)
            throw std::runtime_error("layer " + S(layer_id) + " too narrow to split " + S(n) +
                                     " ways (fan_out " + S(fan_out) + ")");
        for (int k = 0; k < n; ++k) out[k] = Shard{layer_id, devices[k], 0, fan_out, true};
        return out;
    }
    const int q = fan_out / n, r = fan_out % n;
    for (int k = 0, at = 0; k < n; ++k) {
        const int w = q + (k < r);
        out[k] = Shard{layer_id, devices[k], at, at + w, false};
        at += w;
    }
    return out;
}

std::vector<int> split_microbatches(int b, int m) {
    if (b < 1 || m < 1) throw std::invalid_argument("batch and micro-batch count must be >= 1");
    if (m > b)
        throw std::runtime_error("micro-batch smaller than one sample (b=" + S(b) + ", m=" + S(m) + ")");
    std::vector<int> v(m, b / m);
    for (int k = 0; k < b % m; ++k) v[k] += 1;
    return v;
}

void validate_chain(const Chain& g) {
    if (g.L() < 1) throw std::runtime_error("model must have at least one layer");
    for (int i = 0; i < g.L(); ++i) {
        if (g.fan_in[i] < 1 || g.fan_out[i] < 1)
            throw std::runtime_error("layer " + S(i + 1) + ": fan_in and fan_out must be >= 1");
        if (i > 0 && g.fan_out[i - 1] != g.fan_in[i])
            throw std::runtime_error("dimension mismatch between layers " + S(i) + " and " + S(i + 1) +
                                     ": fan_out " + S(g.fan_out[i - 1]) + " vs fan_in " + S(g.fan_in[i]));
    }
}

Plan build_plan(const Chain& g, int n, int Z, bool replicate_narrow) {
    validate_chain(g);
    if (n < 1) throw std::invalid_argument("build_plan: n must be >= 1");
    check_z(g, Z);
    return from_spans(g, spans(g, Z), std::vector<std::vector<int>>(Z, iota1(n)), n, replicate_narrow);
}

Plan build_staged_plan(const Chain& g, const std::vector<std::vector<int>>& groups,
                       bool replicate_narrow) {
    validate_chain(g);
    const int Z = static_cast<int>(groups.size());
    check_z(g, Z);
    int n = 0;
    for (const auto& grp : groups) {
        if (grp.empty()) throw std::invalid_argument("device group must not be empty");
        for (int d : grp) n = d > n ? d : n;
    }
    return from_spans(g, spans(g, Z), groups, n, replicate_narrow);
}

Plan build_plan_with_cuts(const Chain& g, int n, const std::vector<int>& cuts,
                          bool replicate_narrow) {
    validate_chain(g);
    if (n < 1) throw std::invalid_argument("build_plan_with_cuts: n must be >= 1");
    int prev = 0;
    for (int c : cuts) {
        if (c <= prev || c >= g.L()) throw std::runtime_error("invalid span cut at layer " + S(c));
        prev = c;
    }
    return from_spans(g, cuts, std::vector<std::vector<int>>(cuts.size() + 1, iota1(n)), n,
                      replicate_narrow);
}

Plan merge_submodules(const Plan& p, const std::vector<int>& group) {
    if (group.size() < 2) throw std::runtime_error("merge group must have length >= 2");
    for (size_t i = 0; i < group.size(); ++i) {
        if (group[i] < 1 || group[i] > p.Z())
            throw std::runtime_error("merge group index " + S(group[i]) + " out of range 1.." + S(p.Z()));
        if (i > 0 && group[i] != group[i - 1] + 1) throw std::runtime_error("group must be contiguous");
    }
    Plan out = p;
    for (size_t i = 0; i + 1 < group.size(); ++i) out.boundaries[group[i] - 1] = kDirect;
    return out;
}

Plan merge_all(const Plan& p) {
    if (p.Z() < 2) return p;
    return merge_submodules(p, iota1(p.Z()));
}

void validate_plan(const Plan& p, const Chain& g, int cluster_devices) {
    if (p.subs.empty()) throw std::runtime_error("plan has no submodules");
    if (static_cast<int>(p.boundaries.size()) != p.Z() - 1)
        throw std::runtime_error("plan boundary count must be Z-1");
    int expect = 1;
    for (const SubModule& sm : p.subs) {
        if (sm.first_layer != expect || sm.last_layer < sm.first_layer)
            throw std::runtime_error("sub-module spans must partition 1..L in order");
        expect = sm.last_layer + 1;
        if (static_cast<int>(sm.shards.size()) != sm.last_layer - sm.first_layer + 1)
            throw std::runtime_error("sub-module " + S(sm.index) + " missing shard rows");
        for (int l = sm.first_layer; l <= sm.last_layer; ++l) {
            if (l > g.L()) throw std::out_of_range("vector::_M_range_check: layer " + S(l));
            const int fo = g.fan_out[l - 1];
            const auto& sh = sm.layer_shards(l);
            if (sh.size() != sm.devices.size())
                throw std::runtime_error("layer " + S(l) + ": one shard per participating device required");
            if (sh.front().replicated) {
                for (const Shard& s : sh)
                    if (!s.replicated || s.lo != 0 || s.hi != fo)
                        throw std::runtime_error("layer " + S(l) + ": inconsistent replication");
            } else {
                int at = 0;
                for (const Shard& s : sh) {
                    if (s.lo != at || s.hi <= s.lo)
                        throw std::runtime_error("layer " + S(l) + ": shards must tile [0, fan_out) exactly");
                    at = s.hi;
                }
                if (at != fo) throw std::runtime_error("layer " + S(l) + ": shards must tile [0, fan_out) exactly");
            }
            for (size_t i = 0; i < sh.size(); ++i) {
                if (sh[i].device_id != sm.devices[i])
                    throw std::runtime_error("layer " + S(l) + ": shard device order must match sub-module devices");
                if (cluster_devices > 0 && (sh[i].device_id < 1 || sh[i].device_id > cluster_devices))
                    throw std::runtime_error("plan references device " + S(sh[i].device_id) +
                                             " absent from the cluster");
            }
        }
    }
    if (expect != g.L() + 1)
        throw std::runtime_error("plan does not cover all layers (ends at " + S(expect - 1) + " of " +
                                 S(g.L()) + ")");
}

Plan plan_from_flat(const int* f, int len) {
    Plan p;
    int r = 0;
    auto next = [&]() {
        if (r >= len) throw std::invalid_argument("malformed plan encoding (truncated)");
        return f[r++];
    };
    p.n = next();
    const int Z = next();
    if (Z < 1 || Z > 4096) throw std::invalid_argument("malformed plan encoding (Z)");
    for (int j = 0; j < Z; ++j) {
        SubModule sm;
        sm.index = next();
        sm.first_layer = next();
        sm.last_layer = next();
        const int D = next();
        if (D < 1 || D > 4096 || sm.last_layer - sm.first_layer > 1 << 20)
            throw std::invalid_argument("malformed plan encoding (sub-module)");
        for (int d = 0; d < D; ++d) sm.devices.push_back(next());
        for (int l = sm.first_layer; l <= sm.last_layer; ++l) {
            std::vector<Shard> row(D);
            for (int d = 0; d < D; ++d) {
                row[d].layer_id = next();
                row[d].device_id = next();
                row[d].lo = next();
                row[d].hi = next();
                row[d].replicated = next() != 0;
            }
            sm.shards.push_back(std::move(row));
        }
        p.subs.push_back(std::move(sm));
    }
    for (int k = 0; k + 1 < Z; ++k) p.boundaries.push_back(next() ? kDirect : kConcat);
    if (r != len) throw std::invalid_argument("malformed plan encoding (trailing data)");
    return p;
}

std::vector<int> plan_to_flat(const Plan& p) {
    std::vector<int> f{p.n, p.Z()};
    for (const SubModule& sm : p.subs) {
        f.insert(f.end(), {sm.index, sm.first_layer, sm.last_layer, static_cast<int>(sm.devices.size())});
        f.insert(f.end(), sm.devices.begin(), sm.devices.end());
        for (const auto& row : sm.shards)
            for (const Shard& s : row) f.insert(f.end(), {s.layer_id, s.device_id, s.lo, s.hi, s.replicated ? 1 : 0});
    }
    f.insert(f.end(), p.boundaries.begin(), p.boundaries.end());
    return f;
}

}  // namespace ppb
