"""Wave-quantization probe: the same 256 x 2304 GEMM at 74 / 128 / 148 pair tiles (diagnostic:
128 tiles cost ~ the pro-rata share of 148, so stream-K would gain < 1 us here)."""
import ctypes as C, json, os, sys
import torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
from paper_2207_11019_b200 import _lib
from gemm_bench import time_fn
L = _lib.lib(); stream = torch.cuda.current_stream().cuda_stream
for M in (18944, 32768, 37888):
    N, K = 256, 2304
    A = torch.randn(M, K, device="cuda"); B = torch.randn(N, K, device="cuda"); Cc = torch.zeros(M, N, device="cuda")
    def run():
        rc = L.ppb_debug_gemm(C.c_void_p(A.data_ptr()), M, K, K, 0, C.c_void_p(B.data_ptr()), N, K, K, 0, M, N, K, 0,
                              C.c_void_p(Cc.data_ptr()), N, None, 0, None, 0, None, 1.0, None, 0, -256, C.c_void_p(stream))
        _lib.check(rc)
    us = 1000 * time_fn(run, reps=20)
    print(json.dumps({"M": M, "tiles": M // 256, "us": round(us, 1), "tflops": round(2.0 * M * N * K / us / 1e6, 1)}))
