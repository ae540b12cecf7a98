"""Epilogue cost probe: time shard GEMMs with and without the epilogue's global
stores (PPB_GEMM_DBG=2, wrong results), next to cuBLAS TF32 and a plain
write of the same output bytes.  Diagnostic only."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11019_b200 import _lib  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import time_fn  # noqa: E402


def main():
    L = _lib.lib()
    stream = torch.cuda.current_stream().cuda_stream
    torch.backends.cuda.matmul.allow_tf32 = True
    shapes = [(524288, 64, 32), (524288, 64, 576), (131072, 128, 1152), (32768, 256, 2304), (2048, 512, 4608),
              (4096, 8192, 8192)]
    for (M, N, K) in shapes:
        A = torch.randn(M, K, device="cuda")
        B = torch.randn(N, K, device="cuda")
        Cc = torch.zeros(M, N, device="cuda")
        bias = torch.randn(N, device="cuda")
        row = {"M": M, "N": N, "K": K}
        for dbg in ("0", "2"):
            os.environ["PPB_GEMM_DBG"] = dbg
            for bn in (0,):
                def run():
                    rc = L.ppb_debug_gemm(C.c_void_p(A.data_ptr()), M, K, K, 0, C.c_void_p(B.data_ptr()), N, K, K, 0,
                                          M, N, K, 0, C.c_void_p(Cc.data_ptr()), N, C.c_void_p(bias.data_ptr()), 1,
                                          None, 0, None, 1.0, None, 0, bn, C.c_void_p(stream))
                    _lib.check(rc)
                row[f"ppb_dbg{dbg}_us"] = 1000 * time_fn(run, reps=10)
        os.environ["PPB_GEMM_DBG"] = "0"
        row["cublas_us"] = 1000 * time_fn(lambda: torch.matmul(A, B.t()), reps=10)
        row["fill_us"] = 1000 * time_fn(lambda: Cc.fill_(1.0), reps=10)
        row["tflops_ppb"] = 2.0 * M * N * K / row["ppb_dbg0_us"] / 1e6
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
