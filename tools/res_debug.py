"""Per-layer forward check of the residual extension (debug helper)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import cnn_oracle  # noqa: E402
from paper_2207_11019_b200 import api, configs  # noqa: E402
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402

full = len(sys.argv) > 1 and sys.argv[1] == "full"
net = (configs.resnet18_cifar(seed=1) if full else configs.small_resnet(seed=3, hw=8, widths=(8, 16), blocks=(1, 1)))
hw = 32 if full else 8
rng = np.random.default_rng(5)
X = rng.standard_normal((16, hw * hw * 3))
y = rng.integers(0, 10, 16)
ref = cnn_oracle.forward_acts(net, X)
for use_graph in (True,):
    s = api.Session(api.Context([0]), net, 16, api.build_plan(net, 1, 1), 1, UpdateMode.async_per_module,
                    TrainConfig(alpha0=0.0, decay=0.0, iterations=1),
                    PartitionedTrainOptions(multiclass_accuracy=True, use_graph=use_graph))
    s.load_batch(X.astype(np.float32), y)
    s.step(1)
    s.sync()
    for l in range(1, len(net.layers) + 1):
        try:
            g = s.read_tensor(0, l)
        except Exception as e:  # noqa: BLE001
            print(l, "read failed", e)
            continue
        r = ref[l - 1].reshape(16, -1)
        if g.shape != r.shape:
            print(l, "shape", g.shape, r.shape)
            continue
        err = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
        print(f"graph={use_graph} layer {l}: rel {err:.2e}  |g| {np.linalg.norm(g):.3e} |r| {np.linalg.norm(r):.3e}")
    del s
