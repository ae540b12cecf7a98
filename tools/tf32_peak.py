"""Dense TF32 tensor-core peak of this B200, measured the way MEASURED_PEAKS.json
measures bf16 (torch.matmul 8192^3, 2*N^3 FLOPs, CUDA events), with TF32
allowed for fp32 matmuls (cuBLAS picks its tcgen05 kind::tf32 kernels):

  * burst     : best of 10 back-to-back launches (a kernel timed alone)
  * sustained : launches back to back for 4 s (power-capped steady state)

plus the same 8192^3 product on this repo's own tcgen05 GEMM
(ppb_debug_gemm, K-major operands), and the SM clocks / throttle reasons
sampled during each phase.  Prints one JSON object.

    python tools/tf32_peak.py > gpurun_out/tf32_peak.json
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def timed(fn, n):
    import torch

    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def sustained(fn, seconds=4.0):
    import torch

    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k, t0 = 0, time.perf_counter()
    s.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            fn()
        k += 20
        torch.cuda.synchronize()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / k


def main():
    import torch

    from paper_2207_11019_b200 import _lib

    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    N = 8192
    flop = 2.0 * N ** 3
    a = torch.randn(N, N, device="cuda", dtype=torch.float32)
    b = torch.randn(N, N, device="cuda", dtype=torch.float32)
    c = torch.empty(N, N, device="cuda", dtype=torch.float32)
    out = {"what": "dense TF32 (fp32 operands, tensor cores), 8192^3, 2*N^3 FLOPs, CUDA events"}

    def cublas():
        torch.matmul(a, b, out=c)

    for _ in range(3):
        cublas()
    with bench.ClockSampler([0]) as clk:
        ms = timed(cublas, 10)
    out["cublas_tf32_burst_tflops"] = flop / ms / 1e9
    out["cublas_burst_clocks"] = clk.summary()
    with bench.ClockSampler([0], period_s=0.05) as clk:
        ms = sustained(cublas)
    out["cublas_tf32_sustained_tflops"] = flop / ms / 1e9
    out["cublas_sustained_clocks"] = clk.summary()

    L = _lib.lib()
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)

    def ours():
        _lib.check(L.ppb_debug_gemm(C.c_void_p(a.data_ptr()), N, N, N, 0, C.c_void_p(b.data_ptr()), N, N, N, 0,
                                    N, N, N, 0, C.c_void_p(c.data_ptr()), N, None, 0, None, 0, None, 1.0,
                                    C.c_void_p(flag.data_ptr()), 0, 0, None))

    for _ in range(3):
        ours()
    torch.cuda.synchronize()
    with bench.ClockSampler([0]) as clk:
        ms = timed(ours, 10)
    out["ours_tf32_burst_tflops"] = flop / ms / 1e9
    out["ours_burst_clocks"] = clk.summary()
    with bench.ClockSampler([0], period_s=0.05) as clk:
        ms = sustained(ours)
    out["ours_tf32_sustained_tflops"] = flop / ms / 1e9
    out["ours_sustained_clocks"] = clk.summary()
    # cross-check of the product (TF32 rounding: normwise ~1e-3)
    ref = a.double() @ b.double().t()
    out["ours_rel_err"] = float((c.double() - ref).norm() / ref.norm())
    out["gpu"] = torch.cuda.get_device_name(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
