"""Diagnostic: per-layer update error of LeNet-style nets vs the fp64 oracle."""
import sys
import numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from _util import rel_norm  # noqa: E402
import cnn_oracle  # noqa: E402
from paper_2207_11019_b200 import api, configs  # noqa: E402
from paper_2207_11019_b200.api import Batch, PartitionedTrainOptions, TrainConfig, UpdateMode  # noqa: E402


def data(net, b, classes, seed=0):
    rng = np.random.default_rng(seed)
    c = net.layers[0].conv
    return rng.standard_normal((b, c.height, c.width, net.layers[0].in_units())), rng.integers(0, classes, b)


def lenet_implicit(seed):
    rng = np.random.default_rng(seed)
    L = [configs._conv(rng, 1, 6, (32, 32), 5, 2, 2), configs._conv(rng, 6, 16, (16, 16), 5, 2, 2)]
    L += [configs._dense(rng, 16 * 64, 120, 1), configs._dense(rng, 120, 84, 1), configs._dense(rng, 84, 10, 2)]
    return api.TinyNet(L)


for name, mk in [("lenet5", lambda: configs.lenet5(seed=7)), ("implicit", lambda: lenet_implicit(7))]:
    for (n, m, mode) in [(1, 1, 0), (2, 1, 0), (2, 2, 0), (2, 2, 1), (1, 2, 0), (3, 2, 0)]:
        net = mk()
        X, y = data(net, 24, 10)
        plan = api.build_plan(net, n, 1, replicate_narrow=True)
        um = UpdateMode.sync_barrier if mode == 0 else UpdateMode.async_per_module
        r = api.train_partitioned(net, Batch(X, y), TrainConfig(alpha0=0.05, decay=0.01, iterations=1), plan, m, um,
                                  PartitionedTrainOptions(multiclass_accuracy=True), device_map=[0] * n)
        Wr, br, lh, _ = cnn_oracle.train(net, X, y, 0.05, 0.01, 1, m)
        Wg, bg = r.net.pack()
        W0, b0 = net.pack()
        out = []
        o = ob = 0
        for lay in net.layers:
            k, kb = lay.weights.size, lay.bias.size
            out.append((round(rel_norm(Wg[o:o + k] - W0[o:o + k], Wr[o:o + k] - W0[o:o + k]), 4),
                        round(rel_norm(bg[ob:ob + kb] - b0[ob:ob + kb], br[ob:ob + kb] - b0[ob:ob + kb]), 4)))
            o += k
            ob += kb
        print(name, n, m, mode, round(r.loss_history[0] - lh[0], 6), out, flush=True)
