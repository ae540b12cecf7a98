"""F/B overlap of the executed step (north_star (4); reference schedule.cpp:293-296).

One eager step with the streams overlapping as in the CUDA graph
(Session.profile_concurrent: every launch queued behind a spin first, per-op
start / end CUDA events, no serialisation), read with the op structure
(Session.op_meta: micro-batch, plan device, stream role).  Reports, per
micro-batch j, the time during which forward work of micro-batch j+1 runs
concurrently with backward work (input gradients, merges, weight gradients)
of micro-batch j, and the step's per-role busy time.

    python tools/overlap_trace.py [workload] [m] [stash_all|proposed] [n_plan_devices] [Z]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

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


def both(ia, ib):
    return union(ia) + union(ib) - union(ia + ib)


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    mem = sys.argv[3] if len(sys.argv) > 3 else "proposed"
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    Z = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    net, X, y = bench.synthetic_batch(wl, seed=1)
    plan = api.build_plan(net, n, Z)
    s = api.Session(api.Context([0] * n), net, X.shape[0], plan, m, UpdateMode.async_per_module,
                    TrainConfig(iterations=1), PartitionedTrainOptions(multiclass_accuracy=True, pipeline_gate=2,
                                                                       memory_mode=mem))
    s.load_batch(X, y)
    s.step(3)
    s.sync()
    graph_ms = s.time_steps(20) / 20
    s.profile_concurrent(1)
    ops, meta = s.profile_timeline(), s.op_meta()
    recs = []
    for o, mt in zip(ops, meta):
        fwd = mt["role"] == "forward" or (mt["role"] == "main" and o["kind"] == "loss_head")
        recs.append({"kind": o["kind"], "layer": o["layer"], "mb": mt["mb"], "role": mt["role"],
                     "phase": "F" if fwd else ("B" if mt["mb"] >= 0 else "U"),
                     "start": o["start"], "end": o["start"] + o["ms"]})
        print(json.dumps(recs[-1]))
    span = max(r["end"] for r in recs) - min(r["start"] for r in recs)
    iv = lambda ph, j: [(r["start"], r["end"]) for r in recs if r["phase"] == ph and r["mb"] == j]
    overlap = {f"F{j + 2}|B{j + 1}": both(iv("F", j + 1), iv("B", j)) for j in range(m - 1)}
    busy = {ph: union([(r["start"], r["end"]) for r in recs if r["phase"] == ph]) for ph in "FBU"}
    print(json.dumps({"summary": {
        "workload": wl, "m": m, "memory_mode": mem, "plan_devices": n, "Z": Z,
        "eager_concurrent_span_ms": span, "graph_step_ms": graph_ms,
        "sum_op_ms": sum(r["end"] - r["start"] for r in recs),
        "busy_ms_by_phase": busy, "fb_overlap_ms": overlap, "fb_overlap_total_ms": sum(overlap.values()),
        "note": "F = forward ops (incl. loss head) of a micro-batch, B = its input-gradient / merge / per-micro-batch "
                "weight-gradient ops, U = once-per-step updates; device times from CUDA events of one eager step "
                "whose launches were all queued before it ran"}}))


if __name__ == "__main__":
    main()
