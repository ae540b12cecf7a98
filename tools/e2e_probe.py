"""Where the end-to-end step's time goes beyond the device step (diagnostic):
pinned H2D of the batch, load_batch (H2D + input staging), step_host."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_11019_b200 import api  # noqa: E402
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402


def wall(fn, n=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def main():
    w = bench.WORKLOADS["vgg16"]
    net = bench.build_net("vgg16")
    b = w["batch"]
    feat = 32 * 32 * 3
    rng = np.random.default_rng(0)
    Xp = torch.empty((b, feat), dtype=torch.float32, pin_memory=True)
    Xp.numpy()[:] = rng.standard_normal((b, feat), dtype=np.float32)
    yp = torch.empty(b, dtype=torch.int32, pin_memory=True)
    yp.numpy()[:] = rng.integers(0, 10, b)
    Xd = torch.empty((b, feat), device="cuda")
    s = api.Session(api.Context([0]), net, b, api.build_plan(net, 1, 1), 1, UpdateMode.async_per_module,
                    TrainConfig(alpha0=1e-4, decay=1e-2, iterations=1), PartitionedTrainOptions(multiclass_accuracy=True))
    s.load_batch(Xp.numpy(), yp.numpy())
    s.step(3)
    s.sync()
    out = {
        "h2d_pinned_ms": wall(lambda: Xd.copy_(Xp, non_blocking=True)),
        "load_batch_ms": wall(lambda: (s.load_batch(Xp.numpy(), yp.numpy()), s.sync())),
        "device_step_ms": s.time_steps(20) / 20,
        "step_host_ms": wall(lambda: s.step_host(Xp.numpy(), yp.numpy())),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
