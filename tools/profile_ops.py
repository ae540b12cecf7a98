"""Per-op device-time table of one eager step (CUDA events around each op)."""
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
    ops = s.profile_ops()
    tot = sum(o["ms"] for o in ops)
    for o in ops:
        print(json.dumps({**o, "share": o["ms"] / tot}))
    print(json.dumps({"total_ms": tot}))


if __name__ == "__main__":
    main()
