"""VGG-16 eager steps at a given batch (debug helper)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2207_11019_b200 import api, configs  # noqa: E402
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402
b = int(sys.argv[1]) if len(sys.argv) > 1 else 512
net = configs.vgg16_cifar(seed=1)
rng = np.random.default_rng(0)
X = rng.standard_normal((b, 32 * 32 * 3), dtype=np.float32)
y = rng.integers(0, 10, b).astype(np.int32)
s = api.Session(api.Context([0]), net, b, api.build_plan(net, 1, 1), 1, UpdateMode.async_per_module,
                TrainConfig(iterations=1), PartitionedTrainOptions(multiclass_accuracy=True, use_graph=False))
s.load_batch(X, y)
s.step(2)
s.sync()
print("ok", b, s.history()[0])
