"""Network descriptions of the BASELINE.json configurations.

Weights are random-initialised with the reference's rule, uniform
[-0.5, 0.5] / sqrt(fan_in) (tinynet.cpp:176-196), fan_in = ksize^2 * C_in for
conv layers; the RNG is numpy's (synthetic benchmark data,
not the reference's libstdc++ stream — use the oracle's init_net for that).

`init="kaiming"` draws conv / hidden weights from U[-sqrt(6/fan_in),
+sqrt(6/fan_in)] instead (variance 2/fan_in, the ReLU-preserving scale).  The
reference rule has variance 1/(12 fan_in), so every ReLU layer shrinks the
signal variance ~24x: through VGG-16's 13 convs the conv1 gradient ends up
~1e-15 of its weights, below fp32 resolution (the reference trains 2-4 layer
MLPs, where this does not matter).  The benchmarked CNNs use kaiming so the
parity checks at the bench configuration compare real updates of every layer.
"""
from __future__ import annotations

import numpy as np

from .api import ActKind, ConvSpec, TinyLayer, TinyNet


def _scale(fan_in, init):
    # width of the uniform distribution around 0
    return 1.0 / np.sqrt(fan_in) if init == "reference" else 2.0 * np.sqrt(6.0 / fan_in)


def _dense(rng, fi, fo, act, init="reference"):
    s = 1.0 / np.sqrt(fi)
    return TinyLayer((rng.random((fo, fi)) - 0.5) * _scale(fi, init), (rng.random(fo) - 0.5) * s, ActKind(act))


def _conv(rng, cin, cout, hw, k=3, pad=1, pool=1, act=1, init="reference"):
    fan_in = k * k * cin
    s = 1.0 / np.sqrt(fan_in)
    return TinyLayer((rng.random((cout, fan_in)) - 0.5) * _scale(fan_in, init), (rng.random(cout) - 0.5) * s,
                     ActKind(act), ConvSpec(hw[0], hw[1], k, pad, pool))


def dense_net(dims, acts, seed=1) -> TinyNet:
    rng = np.random.default_rng(seed)
    return TinyNet([_dense(rng, dims[l], dims[l + 1], acts[l]) for l in range(len(acts))])


def mlp784(seed=1) -> TinyNet:
    """BASELINE configs[0]: MLP 784-512-512-10."""
    return dense_net([784, 512, 512, 10], [1, 1, 2], seed)


def wide_mlp(seed=1) -> TinyNet:
    """BASELINE configs[4]: 4 layers of 8192 -> 8192."""
    return dense_net([8192] * 5, [1, 1, 1, 2], seed)


VGG16 = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def vgg16_cifar(seed=1, classes=10, widths=VGG16, hw=32, cin=3, init="reference") -> TinyNet:
    """BASELINE configs[2]: VGG-16 on 32x32x3 (13 conv 3x3 + ReLU, 5 max pools,
    classifier 512 -> classes)."""
    rng = np.random.default_rng(seed)
    layers, c, h = [], cin, hw
    i = 0
    while i < len(widths):
        w = widths[i]
        pool = 2 if i + 1 < len(widths) and widths[i + 1] == "M" else 1
        layers.append(_conv(rng, c, w, (h, h), 3, 1, pool, init=init))
        c = w
        h //= pool
        i += 2 if pool == 2 else 1
    layers.append(_dense(rng, c * h * h, classes, 2))
    return TinyNet(layers)


def small_cnn(seed=1, hw=8, cin=3, widths=(16, "M", 32, "M"), classes=10) -> TinyNet:
    """A scaled-down VGG-style net for parity tests."""
    return vgg16_cifar(seed, classes, list(widths), hw, cin)


def lenet5(seed=1, classes=10, hw=28, cin=1, init="reference") -> TinyNet:
    """BASELINE configs[1]: LeNet-5-style CNN on 28x28x1: C1 5x5x6 (pad 2, the
    original's 32x32 input) + ReLU + 2x2 max-pool -> 14x14x6, C3 5x5x16
    (valid) + ReLU + pool -> 5x5x16, F5 400 -> 120, F6 120 -> 84, output
    84 -> classes (softmax).  The 28x28 / 10x10 grids do not tile into
    128-pixel TMA boxes, so both convs run on the generic im2col path."""
    rng = np.random.default_rng(seed)
    layers = [_conv(rng, cin, 6, (hw, hw), 5, 2, 2, init=init), _conv(rng, 6, 16, (hw // 2, hw // 2), 5, 0, 2, init=init)]
    s = (hw // 2 - 4) // 2
    layers += [_dense(rng, 16 * s * s, 120, 1, init), _dense(rng, 120, 84, 1, init), _dense(rng, 84, classes, 2)]
    return TinyNet(layers)


def resnet18_cifar(seed=1, classes=10, hw=32, cin=3, widths=(64, 128, 256, 512), blocks=(2, 2, 2, 2),
                   init="kaiming") -> TinyNet:
    """BASELINE configs[3]: ResNet-18 on 32x32x3 (the CIFAR variant: 3x3 stem,
    17 conv 3x3 + the classifier).  Four stages of two basic blocks (two 3x3
    convs, ReLU after the residual add); each later stage opens with a
    stride-2 conv and its shortcut is ResNet "option A" (every 2nd position,
    channels zero-padded: parameter-free, He et al. 2016 §4.2), the other
    shortcuts are identities; the last conv ends in a global average pool,
    then 512 -> classes.  No batch norm (SURVEY §8d counts conv + fc only:
    3.33 GFLOP / sample)."""
    rng = np.random.default_rng(seed)
    layers = [_conv(rng, cin, widths[0], (hw, hw), init=init)]
    c, h, prev = widths[0], hw, 1
    for st, wd in enumerate(widths):
        for blk in range(blocks[st]):
            down = st > 0 and blk == 0
            la = _conv(rng, c, wd, (h, h), init=init)
            la.conv.stride = 2 if down else 1
            layers.append(la)
            h = h // 2 if down else h
            last = st == len(widths) - 1 and blk == blocks[st] - 1
            lb = _conv(rng, wd, wd, (h, h), pool=h if last else 1, init=init)
            lb.conv.res_from = prev
            lb.conv.pool_avg = last
            layers.append(lb)
            prev, c = len(layers), wd
    layers.append(_dense(rng, c, classes, 2, init))
    return TinyNet(layers)


def small_resnet(seed=1, hw=8, cin=3, widths=(8, 16), blocks=(1, 1), classes=10) -> TinyNet:
    """A scaled-down ResNet for parity tests (identity and option-A
    shortcuts, a stride-2 stage transition, global average pool)."""
    return resnet18_cifar(seed, classes, hw, cin, widths, blocks)
