"""Time the shard GEMM (tcgen05 TF32) against torch/cuBLAS TF32 on one B200.

Prints one JSON line per case: achieved TFLOP/s with CUDA events (warm,
median of reps).  Used to measure the TF32 dense peak (cuBLAS) that the
roofline fractions are quoted against.
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11019_b200 import _lib  # noqa: E402


def time_fn(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    M, N, K = [int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4096, 8192, 8192))]
    flops = 2.0 * M * N * K
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda")
    ms = time_fn(lambda: torch.matmul(a, b.t()))
    print(json.dumps({"case": "torch_tf32_nt", "M": M, "N": N, "K": K, "ms": ms, "tflops": flops / ms / 1e9}))
    L = _lib.lib()
    stream = torch.cuda.current_stream().cuda_stream
    for a_mn, b_mn in [(0, 0), (0, 1), (1, 1)]:
        A = torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, K, device="cuda")
        B = torch.randn(K, N, device="cuda") if b_mn else torch.randn(N, K, device="cuda")
        Cc = torch.empty(M, N, device="cuda")
        for bn in (0, 256, -256, -128):
            def run():
                rc = L.ppb_debug_gemm(C.c_void_p(A.data_ptr()), A.shape[0], A.shape[1], A.shape[1], a_mn,
                                      C.c_void_p(B.data_ptr()), B.shape[0], B.shape[1], B.shape[1], b_mn,
                                      M, N, K, 0, C.c_void_p(Cc.data_ptr()), N, None, 0, None, 0, None,
                                      1.0, None, 0, bn, C.c_void_p(stream))
                _lib.check(rc)
            ms = time_fn(run)
            print(json.dumps({"case": f"ppb_tc a_mn={a_mn} b_mn={b_mn} bn={bn}", "M": M, "N": N, "K": K,
                              "ms": ms, "tflops": flops / ms / 1e9}))


if __name__ == "__main__":
    main()
