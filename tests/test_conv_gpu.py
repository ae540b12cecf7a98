"""Implicit-GEMM convolution products (csrc/conv.h) on the tcgen05 kernel
against PyTorch float64 (torch.nn.functional.conv2d and its input / weight
gradients).  Layouts: padded NHWC activations and error signals, weights in
GEMM layout [u][k*k][ck].  Tolerance: normwise 2e-3 (TF32 operands)."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2207_11019_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def r4(x):
    return (x + 3) // 4 * 4


def r32(x):
    return (x + 31) // 32 * 32


def _setup(N, H, W, Cin, u, k, p, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(N, H, W, Cin, device="cuda", generator=g, dtype=torch.float64)
    wt = torch.randn(u, k, k, Cin, device="cuda", generator=g, dtype=torch.float64) / (k * (Cin ** 0.5))
    Ho, Wo = H + 2 * p - k + 1, W + 2 * p - k + 1
    dy = torch.randn(N, Ho, Wo, u, device="cuda", generator=g, dtype=torch.float64)
    ldx, ldd, ck = r4(Cin), r4(u), r32(Cin)
    x_pad = torch.zeros(N, H + 2 * p, W + 2 * p, ldx, device="cuda")
    x_pad[:, p:p + H, p:p + W, :Cin] = x.float()
    w = torch.zeros(u, k * k, ck, device="cuda")
    w[:, :, :Cin] = wt.reshape(u, k * k, Cin).float()
    q = k - 1 - p
    d_pad = torch.zeros(N, Ho + 2 * q, Wo + 2 * q, ldd, device="cuda")
    d_pad[:, q:q + Ho, q:q + Wo, :u] = dy.float()
    return x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo


def _call(which, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, ldo, bn):
    rc = _lib.lib().ppb_debug_conv(which, C.c_void_p(x_pad.data_ptr()), N, H, W, Cin, ldx, p, k,
                                   C.c_void_p(w.data_ptr()), u, C.c_void_p(d_pad.data_ptr()), ldd,
                                   C.c_void_p(out.data_ptr()), ldo, bn, None)
    _lib.check(rc)
    torch.cuda.synchronize()


def rel(a, b):
    return ((a - b).norm() / b.norm()).item()


SHAPES = [  # N, H, W, Cin, u, k, p  (VGG-16 CIFAR geometries, scaled batch)
    (4, 32, 32, 64, 64, 3, 1),
    (4, 32, 32, 3, 64, 3, 1),
    (8, 16, 16, 64, 128, 3, 1),
    (16, 8, 8, 128, 96, 3, 1),
    (32, 4, 4, 256, 256, 3, 1),
    (64, 2, 2, 512, 160, 3, 1),
    (3, 2, 2, 40, 24, 3, 1),
]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bn", [0, 64, -64, -128])
def test_conv_forward(shape, bn):
    N, H, W, Cin, u, k, p = shape
    x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo = _setup(*shape)
    out = torch.zeros(N * Ho * Wo, r4(u), device="cuda")
    _call(0, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, r4(u), bn)
    ref = torch.nn.functional.conv2d(x.permute(0, 3, 1, 2), wt.permute(0, 3, 1, 2), padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(N * Ho * Wo, u)
    assert rel(out[:, :u].double(), ref) < 2e-3


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bn", [0, -256])
def test_conv_dgrad(shape, bn):
    N, H, W, Cin, u, k, p = shape
    x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo = _setup(*shape, seed=1)
    out = torch.zeros(N * H * W, r4(Cin), device="cuda")
    _call(1, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, r4(Cin), bn)
    ref = torch.nn.grad.conv2d_input((N, Cin, H, W), wt.permute(0, 3, 1, 2), dy.permute(0, 3, 1, 2), padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(N * H * W, Cin)
    assert rel(out[:, :Cin].double(), ref) < 2e-3


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("bn", [0, 128, -256])
def test_conv_wgrad(shape, bn):
    N, H, W, Cin, u, k, p = shape
    x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo = _setup(*shape, seed=2)
    out = torch.zeros(u, k * k * ck, device="cuda")
    _call(2, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, k * k * ck, bn)
    ref = torch.nn.grad.conv2d_weight(x.permute(0, 3, 1, 2), (u, Cin, k, k), dy.permute(0, 3, 1, 2), padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(u, k * k, Cin)
    got = out.reshape(u, k * k, ck)
    assert rel(got[:, :, :Cin].double(), ref) < 2e-3
    assert torch.count_nonzero(got[:, :, Cin:]) == 0


@pytest.mark.parametrize("shape", SHAPES)
def test_conv_wgrad_transposed_splitk(shape):
    """dW^T orientation (M = k*k*ck, N = u) with split-K and the transposed SGD
    epilogue writing W[u][tap][c] (the session uses it for u < 128)."""
    N, H, W, Cin, u, k, p = shape
    x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo = _setup(*shape, seed=3)
    out = torch.zeros(u, k * k * ck, device="cuda")
    _call(3, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, k * k * ck, 0)
    ref = torch.nn.grad.conv2d_weight(x.permute(0, 3, 1, 2), (u, Cin, k, k), dy.permute(0, 3, 1, 2), padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(u, k * k, Cin)
    got = out.reshape(u, k * k, ck)
    assert rel(got[:, :, :Cin].double(), ref) < 2e-3


# Halo-reuse kernel (csrc/conv_halo.cu): padded-position GEMM rows, one halo
# box per 32-channel block shared by the 9 taps.  force = 1000 + bn (1-CTA) or
# 2000 + bn (CTA pair).
HALO_SHAPES = [
    (4, 32, 32, 64, 64, 3, 1),
    (8, 16, 16, 64, 128, 3, 1),
    (3, 16, 32, 96, 80, 3, 1),
    (2, 32, 32, 3, 64, 3, 1),
    (5, 16, 16, 128, 256, 3, 1),
]
HALO_TILES = [1064, 1128, 1256, 2064, 2128, 2256]


@pytest.mark.parametrize("shape", HALO_SHAPES)
@pytest.mark.parametrize("bn", HALO_TILES)
def test_conv_forward_halo(shape, bn):
    test_conv_forward(shape, bn)


@pytest.mark.parametrize("shape", HALO_SHAPES)
@pytest.mark.parametrize("bn", HALO_TILES)
def test_conv_dgrad_halo(shape, bn):
    test_conv_dgrad(shape, bn)


def test_halo_ineligible_is_refused():
    """A 4x4 grid (2.25x padded-space overhead) is not routed to the halo
    kernel; forcing it reports an error instead of computing."""
    shape = (32, 4, 4, 256, 256, 3, 1)
    x, wt, dy, x_pad, w, d_pad, ldx, ldd, ck, Ho, Wo = _setup(*shape)
    N, H, W, Cin, u, k, p = shape
    out = torch.zeros(N * Ho * Wo, r4(u), device="cuda")
    with pytest.raises(Exception):
        _call(0, N, H, W, Cin, ldx, p, k, x_pad, w, u, d_pad, ldd, out, r4(u), 1128)
