// pipeplan_b200: the reference CLI's training-facing subcommands (SPEC.md:503-550,
// the `verify` and `demo` operations; the reference's tools/main.cpp is not in
// the tree) over the B200 drop-in.  pipeplan::train_partitioned here is
// dropin/train_partitioned_b200.cpp (tcgen05 kernels behind the C ABI); every
// other symbol is the reference library compiled from its own sources.
//
//   pipeplan_b200 verify [--seeds N] [--seed S] [--inject-fault] [--out DIR]
//       run_verification (verify.cpp:104-247): exit 0 iff every property
//       passes, 1 on a failure (naming the property), 2 on a usage error.
//   pipeplan_b200 demo [--dims 784,512,512,10] [-n N] [-Z Z] [-m M]
//                      [--update sync|async] [--merge] [--batch B]
//                      [--iterations T] [--seed S] [--out DIR]
//       the paper-default training run (paper §IV.E: batch 6,
//       cross entropy, 50 iterations, alpha 1e-4 decayed by 1e-2) on the
//       synthetic two-class blobs (make_blobs), partitioned over n devices
//       (build_plan(n, Z), optionally merge_all), m micro-batches (default n);
//       writes plan.json and history.csv (iteration, loss, ACC) to DIR and
//       prints the final loss; the same run through train_sequential is
//       reported beside it with the net distance between the two results.
//   pipeplan_b200 plan [--dims ...] -n N [-Z Z] [--merge] [--out DIR]
//       the plan document (serialize_plan) for build_plan(n, Z).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "pipeplan/partition.hpp"
#include "pipeplan/tinynet.hpp"
#include "pipeplan/train_partitioned.hpp"
#include "pipeplan/verify.hpp"

using namespace pipeplan;

namespace {

struct Args {
    std::string cmd;
    std::vector<int> dims{784, 512, 512, 10};
    int n = 2, Z = 1, m = 0, batch = 6, iterations = 50, seeds = 100;
    bool merge = false, fault = false, async = false;
    std::uint64_t seed = 1;
    std::string out = ".";
};

int usage(const char* why) {
    std::fprintf(stderr,
                 "usage error: %s\n"
                 "  pipeplan_b200 verify [--seeds N] [--seed S] [--inject-fault] [--out DIR]\n"
                 "  pipeplan_b200 demo [--dims a,b,...] [-n N] [-Z Z] [-m M] [--update sync|async] [--merge]\n"
                 "                     [--batch B] [--iterations T] [--seed S] [--out DIR]\n"
                 "  pipeplan_b200 plan [--dims a,b,...] -n N [-Z Z] [--merge] [--out DIR]\n",
                 why);
    return 2;
}

bool parse_int(const char* s, long long lo, long long hi, long long* v) {
    char* end = nullptr;
    const long long x = std::strtoll(s, &end, 10);
    if (end == s || *end != '\0' || x < lo || x > hi) return false;
    *v = x;
    return true;
}

// returns 0 on success, else the usage-error exit code (2)
int parse(int argc, char** argv, Args* a) {
    if (argc < 2) return usage("missing subcommand");
    a->cmd = argv[1];
    if (a->cmd != "verify" && a->cmd != "demo" && a->cmd != "plan") return usage("unknown subcommand");
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> const char* { return i + 1 < argc ? argv[++i] : nullptr; };
        long long v = 0;
        if (k == "--merge") {
            a->merge = true;
        } else if (k == "--inject-fault") {
            a->fault = true;
        } else if (k == "--dims") {
            const char* s = val();
            if (!s) return usage("--dims needs a list");
            a->dims.clear();
            std::stringstream ss(s);
            std::string tok;
            while (std::getline(ss, tok, ',')) {
                if (!parse_int(tok.c_str(), 1, 1 << 24, &v)) return usage("bad --dims entry");
                a->dims.push_back(static_cast<int>(v));
            }
            if (a->dims.size() < 2) return usage("--dims needs at least two widths");
        } else if (k == "--update") {
            const char* s = val();
            if (!s || (std::strcmp(s, "sync") != 0 && std::strcmp(s, "async") != 0)) return usage("--update sync|async");
            a->async = std::strcmp(s, "async") == 0;
        } else if (k == "--out") {
            const char* s = val();
            if (!s) return usage("--out needs a directory");
            a->out = s;
        } else {
            const char* s = val();
            if (!s || !parse_int(s, 0, 1LL << 40, &v)) return usage(("bad value for " + k).c_str());
            if (k == "-n") a->n = static_cast<int>(v);
            else if (k == "-Z") a->Z = static_cast<int>(v);
            else if (k == "-m") a->m = static_cast<int>(v);
            else if (k == "--batch") a->batch = static_cast<int>(v);
            else if (k == "--iterations") a->iterations = static_cast<int>(v);
            else if (k == "--seeds") a->seeds = static_cast<int>(v);
            else if (k == "--seed") a->seed = static_cast<std::uint64_t>(v);
            else return usage(("unknown flag " + k).c_str());
        }
    }
    if (a->n < 1) return usage("n must be >= 1");
    if (a->Z < 1) return usage("Z must be >= 1");
    if (a->batch < 1 || a->iterations < 1 || a->seeds < 1) return usage("batch, iterations and seeds must be >= 1");
    return 0;
}

bool write_file(const std::string& dir, const std::string& name, const std::string& text) {
    ::mkdir(dir.c_str(), 0755);
    std::ofstream f(dir + "/" + name);
    f << text;
    return static_cast<bool>(f);
}

TinyNet demo_net(const Args& a) {
    std::vector<ActKind> acts(a.dims.size() - 1, ActKind::relu);
    acts.back() = ActKind::softmax_last;
    return init_net(a.dims, acts, a.seed);
}

PartitionPlan demo_plan(const Args& a, const TinyNet& net) {
    PartitionPlan p = build_plan(model_graph_of(net, "demo"), a.n, a.Z);
    return a.merge ? merge_all(p) : p;
}

int cmd_verify(const Args& a) {
    VerifyOptions o;
    o.seeds = a.seeds;
    if (a.seed != 1) o.base_seed = a.seed;
    o.inject_gradient_fault = a.fault;
    VerifyReport r = run_verification(o);
    // oracle-equivalence is written for the fp64 reference (tol 1e-6); the
    // drop-in trains in fp32 (PPB_PRECISION=fp32) or TF32 tensor-core
    // arithmetic, so that one property is judged at the precision's
    // tolerance (the same bounds tests/test_dropin_gpu.py holds it to)
    const char* prec = std::getenv("PPB_PRECISION");
    const bool fp32 = prec != nullptr && std::strcmp(prec, "fp32") == 0;
    for (PropertyResult& p : r.properties) {
        if (p.name != "oracle-equivalence-sync") continue;
        p.note += (p.note.empty() ? "" : "; ") + std::string("fp64 tolerance ") + std::to_string(p.tolerance) +
                  " relaxed to the " + (fp32 ? "fp32" : "tf32") + " bound";
        p.tolerance = fp32 ? 2e-5 : 5e-3;
        p.pass = p.max_err <= p.tolerance;
    }
    std::printf("%s", verify_report_text(r).c_str());
    write_file(a.out, "verify_report.json", serialize_verify_report(r));
    if (r.all_pass()) return 0;
    for (const PropertyResult& p : r.properties)
        if (!p.pass) std::fprintf(stderr, "FAILED property %s: max_err %.3e > %.1e (%s)\n", p.name.c_str(), p.max_err,
                                  p.tolerance, p.note.c_str());
    return 1;
}

int cmd_plan(const Args& a) {
    const TinyNet net = demo_net(a);
    const PartitionPlan p = demo_plan(a, net);
    const std::string doc = serialize_plan(p);
    std::printf("%s\n", doc.c_str());
    return write_file(a.out, "plan.json", doc) ? 0 : 2;
}

int cmd_demo(const Args& a) {
    const TinyNet net = demo_net(a);
    const Batch batch = make_blobs(a.batch, a.dims.front(), 1.0, a.seed + 12);
    const PartitionPlan plan = demo_plan(a, net);
    TrainConfig cfg;  // paper §IV.E defaults: alpha0 1e-4, decay 1e-2, cross entropy
    cfg.iterations = a.iterations;
    cfg.seed = a.seed;
    const int m = a.m > 0 ? a.m : a.n;
    const TrainResult r =
        train_partitioned(net, batch, cfg, plan, m, a.async ? UpdateMode::async_per_module : UpdateMode::sync_barrier);
    const TrainResult s = train_sequential(net, batch, cfg);
    std::ostringstream csv;
    csv << "iteration,loss,acc\n";
    csv.precision(17);
    for (size_t t = 0; t < r.loss_history.size(); ++t)
        csv << t + 1 << ',' << r.loss_history[t] << ',' << r.acc_history[t] << '\n';
    if (!write_file(a.out, "history.csv", csv.str()) || !write_file(a.out, "plan.json", serialize_plan(plan))) {
        std::fprintf(stderr, "cannot write to %s\n", a.out.c_str());
        return 2;
    }
    std::printf("demo: n=%d Z=%d m=%d %s, batch %d, %d iterations: loss %.6f -> %.6f, ACC %.3f; "
                "train_sequential loss %.6f, net_distance %.3e\n",
                a.n, a.Z, m, a.async ? "async" : "sync", a.batch, a.iterations, r.loss_history.front(),
                r.loss_history.back(), r.acc_history.back(), s.loss_history.back(), net_distance(r.net, s.net));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    if (const int rc = parse(argc, argv, &a)) return rc;
    try {
        if (a.cmd == "verify") return cmd_verify(a);
        if (a.cmd == "plan") return cmd_plan(a);
        return cmd_demo(a);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
