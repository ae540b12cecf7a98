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

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
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

// ------------------------------------------------------------------ JSON I/O

namespace {

std::string jstr(const std::string& v) {
    std::string o = "\"";
    for (char c : v) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            case '\r': o += "\\r"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char buf[8];
                    snprintf(buf, sizeof(buf), "\\u%04x", c);
                    o += buf;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

std::string ind(int d) { return std::string(2 * d, ' '); }

std::string int_array(const std::vector<int>& v) {
    std::string o = "[";
    for (size_t i = 0; i < v.size(); ++i) o += (i ? "," : "") + S(v[i]);
    return o + "]";
}

std::string str_array(const std::vector<std::string>& v, int d) {
    if (v.empty()) return "[]";
    std::string o = "[\n";
    for (size_t i = 0; i < v.size(); ++i) o += ind(d + 1) + jstr(v[i]) + (i + 1 < v.size() ? ",\n" : "\n");
    return o + ind(d) + "]";
}

// Minimal JSON reader for plan documents (objects, arrays, numbers, strings,
// booleans, null).
struct JVal {
    enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
    double num = 0;
    bool b = false;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal* find(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
    const JVal& at(const std::string& k) const {
        const JVal* v = find(k);
        if (!v) throw std::runtime_error("[json.exception.out_of_range.403] key '" + k + "' not found");
        return *v;
    }
    const JVal& at(size_t i) const {
        if (kind != kArr || i >= arr.size())
            throw std::runtime_error("[json.exception.out_of_range.401] array index " + S(static_cast<long long>(i)) +
                                     " is out of range");
        return arr[i];
    }
    int as_int() const {
        if (kind != kNum) throw std::runtime_error("[json.exception.type_error.302] type must be number");
        return static_cast<int>(num);
    }
    const std::string& as_str() const {
        if (kind != kStr) throw std::runtime_error("[json.exception.type_error.302] type must be string");
        return str;
    }
};

struct JParser {
    const std::string& t;
    size_t i = 0;
    explicit JParser(const std::string& s) : t(s) {}
    [[noreturn]] void fail(const std::string& what) {
        throw std::runtime_error("plan parse error: " + what + " at offset " + S(static_cast<long long>(i)));
    }
    void ws() {
        while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\t' || t[i] == '\r')) ++i;
    }
    JVal value() {
        ws();
        if (i >= t.size()) fail("unexpected end of input");
        JVal v;
        const char c = t[i];
        if (c == '{') {
            v.kind = JVal::kObj;
            ++i;
            ws();
            if (i < t.size() && t[i] == '}') {
                ++i;
                return v;
            }
            while (true) {
                ws();
                JVal k = value();
                if (k.kind != JVal::kStr) fail("object key must be a string");
                ws();
                if (i >= t.size() || t[i] != ':') fail("expected ':'");
                ++i;
                v.obj.emplace_back(k.str, value());
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == '}') {
                    ++i;
                    return v;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JVal::kArr;
            ++i;
            ws();
            if (i < t.size() && t[i] == ']') {
                ++i;
                return v;
            }
            while (true) {
                v.arr.push_back(value());
                ws();
                if (i < t.size() && t[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < t.size() && t[i] == ']') {
                    ++i;
                    return v;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::kStr;
            ++i;
            while (i < t.size() && t[i] != '"') {
                if (t[i] == '\\' && i + 1 < t.size()) {
                    const char e = t[i + 1];
                    v.str += e == 'n' ? '\n' : e == 't' ? '\t' : e == 'r' ? '\r' : e;
                    i += 2;
                } else {
                    v.str += t[i++];
                }
            }
            if (i >= t.size()) fail("unterminated string");
            ++i;
            return v;
        }
        if (t.compare(i, 4, "true") == 0) {
            v.kind = JVal::kBool;
            v.b = true;
            i += 4;
            return v;
        }
        if (t.compare(i, 5, "false") == 0) {
            v.kind = JVal::kBool;
            i += 5;
            return v;
        }
        if (t.compare(i, 4, "null") == 0) {
            i += 4;
            return v;
        }
        size_t end = i;
        while (end < t.size() && (isdigit(static_cast<unsigned char>(t[end])) || t[end] == '-' || t[end] == '+' ||
                                  t[end] == '.' || t[end] == 'e' || t[end] == 'E'))
            ++end;
        if (end == i) fail("syntax error");
        v.kind = JVal::kNum;
        v.num = std::stod(t.substr(i, end - i));
        i = end;
        return v;
    }
};

}  // namespace

std::string serialize_plan(const Plan& p, const std::vector<std::string>& provenance) {
    std::vector<std::string> bounds;
    for (int b : p.boundaries) bounds.push_back(b == kConcat ? "concat" : "direct");
    std::string o = "{\n";
    o += ind(1) + "\"boundaries\": " + str_array(bounds, 1) + ",\n";
    o += ind(1) + "\"n\": " + S(p.n) + ",\n";
    o += ind(1) + "\"provenance\": " + str_array(provenance, 1) + ",\n";
    o += ind(1) + "\"schema\": 1,\n";
    o += ind(1) + "\"submodules\": ";
    if (p.subs.empty()) {
        o += "[]\n";
    } else {
        o += "[\n";
        for (size_t j = 0; j < p.subs.size(); ++j) {
            const SubModule& sm = p.subs[j];
            o += ind(2) + "{\n";
            o += ind(3) + "\"devices\": " + int_array(sm.devices) + ",\n";
            std::vector<const Shard*> all;
            for (const auto& row : sm.shards)
                for (const Shard& s : row) all.push_back(&s);
            o += ind(3) + "\"shards\": ";
            if (all.empty()) {
                o += "[]";
            } else {
                o += "[\n";
                for (size_t k = 0; k < all.size(); ++k) {
                    const Shard& s = *all[k];
                    o += ind(4) + "{\n";
                    o += ind(5) + "\"device\": " + S(s.device_id) + ",\n";
                    o += ind(5) + "\"layer\": " + S(s.layer_id) + ",\n";
                    o += ind(5) + "\"range\": " + int_array({s.lo, s.hi});
                    o += s.replicated ? ",\n" + ind(5) + "\"replicated\": true\n" : "\n";
                    o += ind(4) + "}" + (k + 1 < all.size() ? ",\n" : "\n");
                }
                o += ind(3) + "]";
            }
            o += ",\n" + ind(3) + "\"span\": " + int_array({sm.first_layer, sm.last_layer}) + "\n";
            o += ind(2) + "}" + (j + 1 < p.subs.size() ? ",\n" : "\n");
        }
        o += ind(1) + "]\n";
    }
    return o + "}\n";
}

Plan parse_plan(const std::string& text, std::vector<std::string>* provenance) {
    JParser jp(text);
    const JVal doc = jp.value();
    jp.ws();
    if (jp.i != text.size()) jp.fail("trailing characters");
    Plan p;
    p.n = doc.at("n").as_int();
    int index = 1;
    const JVal& subs = doc.at("submodules");
    for (const JVal& jm : subs.arr) {
        SubModule sm;
        sm.index = index++;
        sm.first_layer = jm.at("span").at(0).as_int();
        sm.last_layer = jm.at("span").at(1).as_int();
        if (const JVal* d = jm.find("devices"))
            for (const JVal& x : d->arr) sm.devices.push_back(x.as_int());
        sm.shards.assign(std::max(0, sm.last_layer - sm.first_layer + 1), {});
        for (const JVal& js : jm.at("shards").arr) {
            Shard s;
            s.layer_id = js.at("layer").as_int();
            s.device_id = js.at("device").as_int();
            s.lo = js.at("range").at(0).as_int();
            s.hi = js.at("range").at(1).as_int();
            const JVal* r = js.find("replicated");
            s.replicated = r != nullptr && r->kind == JVal::kBool && r->b;
            if (s.layer_id < sm.first_layer || s.layer_id > sm.last_layer)
                throw std::runtime_error("plan shard layer " + S(s.layer_id) + " outside its sub-module span");
            sm.shards[s.layer_id - sm.first_layer].push_back(s);
        }
        if (sm.devices.empty() && !sm.shards.empty())
            for (const Shard& s : sm.shards.front()) sm.devices.push_back(s.device_id);
        p.subs.push_back(std::move(sm));
    }
    for (const JVal& jb : doc.at("boundaries").arr) {
        const std::string& b = jb.as_str();
        if (b == "concat") p.boundaries.push_back(kConcat);
        else if (b == "direct") p.boundaries.push_back(kDirect);
        else throw std::runtime_error("unknown boundary kind \"" + b + "\"");
    }
    if (provenance) {
        provenance->clear();
        if (const JVal* pv = doc.find("provenance"))
            for (const JVal& x : pv->arr) provenance->push_back(x.as_str());
    }
    return p;
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
