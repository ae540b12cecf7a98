"""Kernel-level tests of the shard GEMM (tcgen05 TF32 and exact-fp32 SIMT)
against a plain PyTorch fp64 reference of the same product.

C[m][n] = sum_k A(m,k) B(n,k); operands K-major or MN-major (csrc/gemm.h).
Tolerances: TF32 inputs carry 10 explicit mantissa bits, so against a
reference computed on TF32-truncated inputs the remaining error is fp32
accumulation only (normwise <= 1e-5); against full-precision inputs it is
<= 2e-3 normwise.  The fp32 SIMT path is <= 1e-5 normwise.
"""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2207_11019_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def _padded(rows, cols, gen, scale=1.0):
    ld = (cols + 3) // 4 * 4
    base = torch.empty(rows, ld, device="cuda", dtype=torch.float32)
    base.normal_(generator=gen)
    base.mul_(scale)
    return base, ld


def _tf32_trunc(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def _run(M, N, K, a_mn, b_mn, mode=0, precision=0, force_bn=0, bias=False, relu=False, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    a_base, lda = _padded(K if a_mn else M, M if a_mn else K, gen)
    b_base, ldb = _padded(K if b_mn else N, N if b_mn else K, gen)
    A = a_base[:, : (M if a_mn else K)]
    B = b_base[:, : (N if b_mn else K)]
    Am = A.t() if a_mn else A  # (M, K)
    Bm = B.t() if b_mn else B  # (N, K)
    ldc = (N + 3) // 4 * 4
    c_base = torch.zeros(M, ldc, device="cuda", dtype=torch.float32)
    bias_t = torch.randn(N, device="cuda", generator=gen) if bias else None
    mask_t = None
    alpha = None
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    if mode == 1:
        mask_t = torch.randn(M, ldc, device="cuda", generator=gen)
    if mode == 2:
        c_base.normal_(generator=gen)
        alpha = torch.tensor([0.25], device="cuda", dtype=torch.float64)
    c_before = c_base.clone()
    L = _lib.lib()
    rc = L.ppb_debug_gemm(
        C.c_void_p(a_base.data_ptr()), a_base.shape[0], A.shape[1], lda, int(a_mn),
        C.c_void_p(b_base.data_ptr()), b_base.shape[0], B.shape[1], ldb, int(b_mn),
        M, N, K, mode, C.c_void_p(c_base.data_ptr()), ldc,
        C.c_void_p(bias_t.data_ptr()) if bias_t is not None else None, int(relu),
        C.c_void_p(mask_t.data_ptr()) if mask_t is not None else None, ldc,
        C.c_void_p(alpha.data_ptr()) if alpha is not None else None, 0.5,
        C.c_void_p(flag.data_ptr()), precision, force_bn, None)
    _lib.check(rc)
    torch.cuda.synchronize()

    def ref(a, b):
        r = a.double() @ b.double().t()
        if mode == 0:
            if bias_t is not None:
                r = r + bias_t.double()
            if relu:
                r = r.clamp_min(0)
        elif mode == 1:
            r = r * (mask_t[:, :N].double() > 0)
        elif mode == 2:
            r = c_before[:, :N].double() - 0.25 * (r * 0.5)
        return r

    out = c_base[:, :N].double()
    full = ref(Am, Bm)
    trunc = ref(_tf32_trunc(Am.contiguous()), _tf32_trunc(Bm.contiguous()))
    nf = full.norm().item() or 1.0
    err_full = (out - full).norm().item() / nf
    err_trunc = (out - trunc).norm().item() / (trunc.norm().item() or 1.0)
    # padding columns must be untouched
    if ldc > N:
        assert torch.equal(c_base[:, N:], c_before[:, N:])
    return err_full, err_trunc, flag.item()


SHAPES = [(128, 256, 64), (300, 200, 100), (64, 5, 512), (7, 3, 5), (1000, 520, 777), (256, 1024, 2048)]
MAJORS = [(False, False), (False, True), (True, True), (True, False)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("majors", MAJORS)
def test_tc_gemm_store(shape, majors):
    M, N, K = shape
    ef, et, _ = _run(M, N, K, *majors)
    assert ef < 2e-3, (ef, et)
    assert et < 1e-4, (ef, et)


@pytest.mark.parametrize("bn", [64, 128, 256, -64, -128, -256])
def test_tc_gemm_tile_widths(bn):
    """1-CTA tiles (bn > 0) and CTA-pair cta_group::2 tiles (bn < 0)."""
    ef, et, _ = _run(640, 700, 300, False, True, force_bn=bn, bias=True, relu=True)
    assert ef < 2e-3 and et < 1e-4, (ef, et)


@pytest.mark.parametrize("majors", MAJORS)
@pytest.mark.parametrize("shape", [(1000, 520, 777), (300, 260, 64), (2048, 1024, 512)])
@pytest.mark.parametrize("bn", [-64, -128, -256])
def test_tc_gemm_pair_majors(majors, shape, bn):
    ef, et, _ = _run(*shape, *majors, force_bn=bn)
    assert ef < 2e-3 and et < 1e-4, (ef, et)


@pytest.mark.parametrize("bn", [-256, 256, -64])
def test_gemm_sgd_epilogue_pairs(bn):
    ef, _, flag = _run(520, 600, 256, True, True, mode=2, force_bn=bn)
    assert ef < 2e-3 and flag == 0


@pytest.mark.parametrize("majors", MAJORS)
def test_simt_gemm_exact(majors):
    ef, et, _ = _run(300, 200, 100, *majors, precision=1, bias=True)
    assert ef < 1e-5, ef


@pytest.mark.parametrize("precision", [0, 1])
def test_gemm_mask_and_sgd_epilogues(precision):
    ef, _, _ = _run(200, 300, 96, False, True, mode=1, precision=precision)
    assert ef < 2e-3
    ef, _, flag = _run(300, 260, 128, True, True, mode=2, precision=precision)
    assert ef < 2e-3 and flag == 0


def test_tc_gemm_large():
    ef, et, _ = _run(2048, 4096, 4096, False, False, seed=3)
    assert ef < 2e-3 and et < 1e-4, (ef, et)


@pytest.mark.parametrize("shape", [(64, 96, 65536), (200, 130, 20000), (8, 300, 4096)])
@pytest.mark.parametrize("majors", MAJORS)
def test_tc_gemm_splitk(shape, majors):
    """Few output tiles, long K: the K loop is split and reduced in order."""
    ef, et, _ = _run(*shape, *majors)
    assert ef < 2e-3 and et < 1e-4, (ef, et)
