"""Eager per-op timeline of one VGG-16 step (start, duration, stream) and the
busy/idle structure: union of op intervals vs the step span.  Diagnostic."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2207_11019_b200 import api  # noqa: E402
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    w = bench.WORKLOADS[wl]
    net = bench.build_net(wl)
    c = net.layers[0].conv
    feat = net.layers[0].in_units() * (c.height * c.width if c else 1)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((w["batch"], feat), dtype=np.float32)
    y = rng.integers(0, w["classes"], w["batch"]).astype(np.int32)
    s = api.Session(api.Context([0]), net, w["batch"], api.build_plan(net, 1, 1), 1, UpdateMode.async_per_module,
                    TrainConfig(iterations=1), PartitionedTrainOptions(multiclass_accuracy=True))
    s.load_batch(X, y)
    s.step(3)
    s.sync()
    s.profile(1)
    ops = s.profile_timeline()
    for o in ops:
        print(json.dumps({k: o[k] for k in ("kind", "layer", "stream", "start", "ms")}))
    iv = sorted((o["start"], o["start"] + o["ms"]) for o in ops)
    busy, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                busy += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    busy += cur[1] - cur[0]
    span = max(b for _, b in iv) - min(a for a, _ in iv)
    print(json.dumps({"span_ms": span, "busy_ms": busy, "sum_ms": sum(o["ms"] for o in ops)}))


if __name__ == "__main__":
    main()
