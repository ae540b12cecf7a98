"""Partitioned training of nets with conv layers (BASELINE CNN configs) on the
GPU against the float64 PyTorch restatement oracle/cnn_oracle.py.

Parity for conv is unpinned by the reference (it has no conv); the oracle
follows the reference's partitioned-step semantics on the conv extension.
Tolerance (TF32 operands, fp32 accumulation): net_distance <= 5e-3, loss
|diff| <= 5e-3 * max(1, |ref|).
"""
import numpy as np
import pytest

from _util import net_distance, rel_norm  # noqa: I001  (puts oracle/ on sys.path)
import cnn_oracle  # oracle/cnn_oracle.py (test infrastructure)
from paper_2207_11019_b200 import api, configs
from paper_2207_11019_b200.api import Batch, PartitionedTrainOptions, TrainConfig, UpdateMode

pytestmark = pytest.mark.gpu

TOL = 5e-3


def data(net, b, classes, seed=0):
    rng = np.random.default_rng(seed)
    c = net.layers[0].conv
    X = rng.standard_normal((b, c.height, c.width, net.layers[0].in_units()))
    y = rng.integers(0, classes, b)
    return X, y


NETS = {
    "pool_pool": lambda: configs.small_cnn(3, 8, 3, (16, "M", 32, "M")),
    "nopool_pool": lambda: configs.small_cnn(4, 8, 3, (8, 16, "M")),
    "relayout": lambda: configs.small_cnn(5, 4, 3, (8,)),
    "deep": lambda: configs.small_cnn(6, 16, 5, (16, 16, "M", 32, "M", 48, "M", 64, "M")),
    # BASELINE configs[1]: both convs on the generic im2col path (28x28 / 10x10 grids)
    "lenet5": lambda: configs.lenet5(seed=7),
}


@pytest.mark.parametrize("name", sorted(NETS))
@pytest.mark.parametrize("n,Z,m", [(1, 1, 1), (2, 1, 2), (2, 2, 1), (3, 1, 3)])
def test_cnn_partitioned_matches_oracle(name, n, Z, m):
    net = NETS[name]()
    Z = min(Z, net.num_layers())
    X, y = data(net, 24, 10)
    cfg = TrainConfig(alpha0=0.05, decay=0.01, iterations=3)
    plan = api.build_plan(net, n, Z, replicate_narrow=True)
    r = api.train_partitioned(net, Batch(X, y), cfg, plan, m, UpdateMode.sync_barrier,
                              PartitionedTrainOptions(multiclass_accuracy=True), device_map=[0] * n)
    W0, b0 = net.pack()
    Wr, br, lh, ah = cnn_oracle.train(net, X, y, 0.05, 0.01, 3, m)
    Wg, bg = r.net.pack()
    d = net_distance(Wg, bg, Wr, br)
    assert d <= TOL, d
    for got, ref in zip(r.loss_history, lh):
        assert abs(got - ref) <= TOL * max(1.0, abs(ref)), (got, ref)
    # the update itself (LeNet's C1 sums 24 x 784 pixel products with heavy
    # cancellation: TF32 leaves ~4% on that layer's update even at n = 1)
    assert rel_norm(Wg - W0, Wr - W0) <= (5e-2 if name == "lenet5" else 3e-2)
    assert np.allclose(r.acc_history, ah, atol=2.0 / 24)


def test_cnn_activations_and_error_signal():
    net = NETS["pool_pool"]()
    X, y = data(net, 16, 10, seed=3)
    ctx = api.Context([0, 0])
    plan = api.build_plan(net, 2, 1)
    s = api.Session(ctx, net, 16, plan, 1, UpdateMode.sync_barrier, TrainConfig(alpha0=0.0, decay=0.0, iterations=1),
                    PartitionedTrainOptions(multiclass_accuracy=True))
    s.load_batch(X, y)
    s.step(1)
    ref = cnn_oracle.forward_acts(net, X.reshape(16, -1))
    for l in (1, 2):
        assert rel_norm(s.read_tensor(0, l), ref[l - 1]) <= 2e-3, l


def test_cnn_sync_async_and_microbatch_bitwise():
    net = NETS["deep"]()
    X, y = data(net, 16, 10, seed=4)
    cfg = TrainConfig(alpha0=0.05, decay=0.01, iterations=2)
    plan = api.build_plan(net, 2, 2)
    o = PartitionedTrainOptions(multiclass_accuracy=True)
    a = api.train_partitioned(net, Batch(X, y), cfg, plan, 1, UpdateMode.sync_barrier, o, device_map=[0, 0])
    b = api.train_partitioned(net, Batch(X, y), cfg, plan, 1, UpdateMode.async_per_module, o, device_map=[0, 0])
    c = api.train_partitioned(net, Batch(X, y), cfg, plan, 4, UpdateMode.sync_barrier, o, device_map=[0, 0])
    for r in (b, c):
        assert np.array_equal(a.net.pack()[0], r.net.pack()[0])
        assert a.loss_history == r.loss_history


def test_vgg16_one_step_small_batch():
    """Full VGG-16 (CIFAR) architecture, batch 8, n=2: one step vs the oracle."""
    net = configs.vgg16_cifar(seed=7)
    X, y = data(net, 8, 10, seed=5)
    cfg = TrainConfig(alpha0=0.01, decay=0.0, iterations=1)
    plan = api.build_plan(net, 2, 1)
    r = api.train_partitioned(net, Batch(X, y), cfg, plan, 1, UpdateMode.async_per_module,
                              PartitionedTrainOptions(multiclass_accuracy=True), device_map=[0, 0])
    W0, _ = net.pack()
    Wr, br, lh, _ = cnn_oracle.train(net, X, y, 0.01, 0.0, 1, 1)
    Wg, bg = r.net.pack()
    assert abs(r.loss_history[0] - lh[0]) <= TOL * max(1.0, lh[0])
    assert net_distance(Wg, bg, Wr, br) <= TOL
    assert rel_norm(Wg - W0, Wr - W0) <= 5e-2


def test_vgg16_one_step_n1_halo_fused_merge():
    """n = 1: the 32x32 / 16x16 convs run on the halo kernel and every backward
    merge is fused into the dgrad epilogue (EPI_MERGE)."""
    net = configs.vgg16_cifar(seed=11)
    X, y = data(net, 6, 10, seed=6)
    cfg = TrainConfig(alpha0=0.01, decay=0.0, iterations=2)
    plan = api.build_plan(net, 1, 1)
    r = api.train_partitioned(net, Batch(X, y), cfg, plan, 2, UpdateMode.async_per_module,
                              PartitionedTrainOptions(multiclass_accuracy=True), device_map=[0])
    W0, _ = net.pack()
    Wr, br, lh, _ = cnn_oracle.train(net, X, y, 0.01, 0.0, 2, 2)
    Wg, bg = r.net.pack()
    for got, ref in zip(r.loss_history, lh):
        assert abs(got - ref) <= TOL * max(1.0, abs(ref)), (got, ref)
    assert net_distance(Wg, bg, Wr, br) <= TOL
    assert rel_norm(Wg - W0, Wr - W0) <= 5e-2


@pytest.mark.parametrize("name", ["pool_pool", "nopool_pool", "deep"])
def test_fused_merge_matches_unfused(name, monkeypatch):
    """The fused single-contributor merge produces the same error signals as
    the slot + conv_merge path (only the bias-gradient summation tree differs)."""
    net = NETS[name]()
    X, y = data(net, 12, 10, seed=8)
    cfg = TrainConfig(alpha0=0.05, decay=0.01, iterations=2)
    plan = api.build_plan(net, 1, 1)
    o = PartitionedTrainOptions(multiclass_accuracy=True)
    a = api.train_partitioned(net, Batch(X, y), cfg, plan, 2, UpdateMode.sync_barrier, o, device_map=[0])
    monkeypatch.setenv("PPB_NO_FUSED_MERGE", "1")
    b = api.train_partitioned(net, Batch(X, y), cfg, plan, 2, UpdateMode.sync_barrier, o, device_map=[0])
    Wa, ba = a.net.pack()
    Wb, bb = b.net.pack()
    assert net_distance(Wa, ba, Wb, bb) <= 1e-5
    for p, q in zip(a.loss_history, b.loss_history):
        assert abs(p - q) <= 1e-5 * max(1.0, abs(q))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_lenet5_partitioned_matches_oracle(n):
    """BASELINE configs[1] (LeNet-5-style, 28x28x1, 5x5 convs): plans over 1/2/4
    devices (C1's 6 channels split 2/2/1/1 at n = 4), two micro-batches."""
    net = configs.lenet5(seed=3)
    X, y = data(net, 32, 10, seed=9)
    cfg = TrainConfig(alpha0=0.05, decay=0.01, iterations=3)
    plan = api.build_plan(net, n, 1)
    r = api.train_partitioned(net, Batch(X, y), cfg, plan, 2, UpdateMode.async_per_module,
                              PartitionedTrainOptions(multiclass_accuracy=True), device_map=[0] * n)
    W0, _ = net.pack()
    Wr, br, lh, _ = cnn_oracle.train(net, X, y, 0.05, 0.01, 3, 2)
    Wg, bg = r.net.pack()
    for got, ref in zip(r.loss_history, lh):
        assert abs(got - ref) <= TOL * max(1.0, abs(ref)), (got, ref)
    assert net_distance(Wg, bg, Wr, br) <= TOL
    assert rel_norm(Wg - W0, Wr - W0) <= 5e-2


def _lenet_implicit(seed):
    """LeNet-style net on 32x32 inputs (both convs on the implicit path) with
    dense shards whose boundaries (120 -> 60/60, 84 -> 42/42) fall inside
    32-byte sectors."""
    rng = np.random.default_rng(seed)
    layers = [configs._conv(rng, 1, 6, (32, 32), 5, 2, 2), configs._conv(rng, 6, 16, (16, 16), 5, 2, 2)]
    layers += [configs._dense(rng, 16 * 64, 120, 1), configs._dense(rng, 120, 84, 1), configs._dense(rng, 84, 10, 2)]
    return api.TinyNet(layers)


@pytest.mark.parametrize("m", [1, 2])
def test_unaligned_shard_boundaries_per_layer_update(m):
    """Regression: concurrent shard GEMMs storing column ranges that share a
    32 B sector (TMA bulk stores must not be used there).  Per-layer update
    error against the oracle, n = 2 vs n = 1."""
    errs = {}
    for n in (1, 2):
        net = _lenet_implicit(7)
        X, y = data(net, 24, 10)
        plan = api.build_plan(net, n, 1)
        r = api.train_partitioned(net, Batch(X, y), TrainConfig(alpha0=0.05, decay=0.01, iterations=1), plan, m,
                                  UpdateMode.sync_barrier, PartitionedTrainOptions(multiclass_accuracy=True),
                                  device_map=[0] * n)
        Wr, br, _, _ = cnn_oracle.train(net, X, y, 0.05, 0.01, 1, m)
        Wg, bg = r.net.pack()
        W0, b0 = net.pack()
        e, o = [], 0
        for lay in net.layers:
            k = lay.weights.size
            e.append(rel_norm(Wg[o:o + k] - W0[o:o + k], Wr[o:o + k] - W0[o:o + k]))
            o += k
        errs[n] = e
    for a, b in zip(errs[1], errs[2]):
        assert b <= 1.2 * a + 1e-3, (errs[1], errs[2])
    assert errs[2][-1] <= 5e-3  # head update: TF32-level


def test_lenet5_error_signal_matches_oracle():
    """The generic path's unpadded error signals (col2im + merge) against
    autograd of the fp64 oracle at the conv layers."""
    import torch

    net = configs.lenet5(seed=5)
    X, y = data(net, 8, 10, seed=2)
    ctx = api.Context([0, 0])
    plan = api.build_plan(net, 2, 1)
    s = api.Session(ctx, net, 8, plan, 1, UpdateMode.sync_barrier, TrainConfig(alpha0=0.0, decay=0.0, iterations=1),
                    PartitionedTrainOptions(multiclass_accuracy=True))
    s.load_batch(X, y)
    s.step(1)
    ref = cnn_oracle.forward_acts(net, X.reshape(8, -1))
    for l in (1, 2, 3):  # TF32 operands: error grows ~1e-3 per conv / dense layer
        assert rel_norm(s.read_tensor(0, l), ref[l - 1]) <= 1e-3 * (l + 1), l
    d1 = s.read_tensor(2, 1)  # error signal of C1 (pre-pool grid, channels of device 1's shard)
    assert np.isfinite(d1).all() and np.abs(d1).sum() > 0
    del torch
