// Executed schedule vs the reference's simulator.
//
// Reads a request (JSON, argv[1]) with the plan the B200 executor ran, its
// micro-batch count and the per-task device times MEASURED on the B200
// (tools/sim_crosscheck.py: CUDA events around every op of one serialised
// step, summed per (sub-module, micro-batch) and per boundary transfer), and
// runs the reference's own scheduler and simulator on them, compiled unchanged
// from its sources: build_schedule (schedule.cpp:207-330, pipelined, the
// F(i,j) <- B(i,j-2) gate at :293-296), attach_updates (:332-371),
// simulate (simulate.cpp:159-283) under both memory policies and
// memory_compare (:290-298).  Prints the predicted makespan, per-device busy
// time and peak memory, the proposed / stash_all memory ratio, the number of
// micro-batches each module holds at its peak, and each device's task order
// (kind, module, micro-batch) for comparison with the executor's enqueue
// order.
//
//   request = {"model": <serialize_model document>, "plan": <serialize_plan document>,
//              "m": m, "tf": [[Z x m]], "tb": [[Z x m]], "tcomm": [[(Z-1) x m]],
//              "samples_per_microbatch": s, "bytes_per_param": 4}
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "pipeplan/cost.hpp"
#include "pipeplan/model.hpp"
#include "pipeplan/partition.hpp"
#include "pipeplan/schedule.hpp"
#include "pipeplan/simulate.hpp"

using namespace pipeplan;
using nlohmann::json;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <request.json>\n", argv[0]);
        return 2;
    }
    try {
        std::ifstream in(argv[1]);
        std::stringstream ss;
        ss << in.rdbuf();
        const json req = json::parse(ss.str());
        const ModelGraph g = parse_model(req.at("model").dump());
        const PartitionPlan plan = parse_plan(req.at("plan").dump());
        const int m = req.at("m").get<int>();
        TaskCostTable t;
        t.m = m;
        t.tf = req.at("tf").get<std::vector<std::vector<double>>>();
        t.tb = req.at("tb").get<std::vector<std::vector<double>>>();
        t.tcomm = req.value("tcomm", std::vector<std::vector<double>>{});
        while (static_cast<int>(t.tcomm.size()) < plan.num_submodules() - 1) t.tcomm.emplace_back(m, 0.0);
        SimOptions so;
        so.samples_per_microbatch = req.value("samples_per_microbatch", 1.0);
        so.bytes_per_param = req.value("bytes_per_param", 4.0);
        const Schedule s = attach_updates(build_schedule(plan, m, SchedulePolicy::pipelined),
                                          UpdateMode::async_per_module);
        const SimReport p = simulate(s, t, MemoryMode::proposed, g, plan, so);
        const SimReport a = simulate(s, t, MemoryMode::stash_all, g, plan, so);
        json out;
        out["makespan_s"] = p.makespan_s;
        out["makespan_stash_all_s"] = a.makespan_s;
        out["busy_s"] = p.busy_s;
        out["utilization"] = p.utilization;
        out["peak_mem_bytes_proposed"] = p.peak_mem_bytes;
        out["peak_mem_bytes_stash_all"] = a.peak_mem_bytes;
        out["memory_ratio"] = memory_compare(g, plan, s, t, so);
        // peak stash in micro-batches per module: replay the proposed trace
        std::vector<int> live(static_cast<size_t>(plan.num_submodules()), 0), peak = live;
        std::vector<std::pair<double, int>> ev;  // (time, +module for F start / -module for B end)
        for (const TaskEvent& e : p.trace) {
            const Task& tk = s.dag.nodes[static_cast<size_t>(e.node)];
            if (tk.kind == TaskKind::forward) ev.emplace_back(e.start, tk.module);
            if (tk.kind == TaskKind::backward) ev.emplace_back(e.end, -tk.module);
        }
        std::stable_sort(ev.begin(), ev.end(), [](const auto& x, const auto& y) {
            return x.first < y.first || (x.first == y.first && x.second < y.second);  // frees first
        });
        for (const auto& [time, mod] : ev) {
            const size_t i = static_cast<size_t>(std::abs(mod) - 1);
            live[i] += mod > 0 ? 1 : -1;
            peak[i] = std::max(peak[i], live[i]);
        }
        out["peak_live_microbatches"] = peak;
        json order = json::array();
        for (const auto& lst : s.device_lists) {
            json d = json::array();
            for (int node : lst) {
                const Task& tk = s.dag.nodes[static_cast<size_t>(node)];
                const char* k = tk.kind == TaskKind::forward ? "F" : tk.kind == TaskKind::backward ? "B"
                               : tk.kind == TaskKind::update ? "U" : "C";
                d.push_back(json::array({k, tk.module, tk.microbatch}));
            }
            order.push_back(d);
        }
        out["device_order"] = order;
        std::printf("%s\n", out.dump().c_str());
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
