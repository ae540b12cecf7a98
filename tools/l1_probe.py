"""Pipeline probe on a one-K-block GEMM (VGG conv1 im2col shape): tile shape x
timing-probe bits (PPB_GEMM_DBG: 2 no stores, 4 no epilogue, 8 no MMAs).
Diagnostic only (probe runs produce wrong results)."""
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
    shapes = [(524288, 64, 32), (524288, 64, 128), (32768, 256, 2304)]
    for (M, N, K) in shapes:
        A = torch.randn(M, K, device="cuda")
        B = torch.randn(N, K, device="cuda")
        Cc = torch.zeros(M, N, device="cuda")
        bias = torch.randn(N, device="cuda")
        for bn in (0, 64, 128, -128, -256):
            row = {"M": M, "N": N, "K": K, "bn": bn}
            for dbg in ("0", "2", "4", "12", "8"):
                os.environ["PPB_GEMM_DBG"] = dbg

                def run():
                    rc = L.ppb_debug_gemm(C.c_void_p(A.data_ptr()), M, K, K, 0, C.c_void_p(B.data_ptr()), N, K, K, 0,
                                          M, N, K, 0, C.c_void_p(Cc.data_ptr()), N, C.c_void_p(bias.data_ptr()), 1,
                                          None, 0, None, 1.0, None, 0, bn, C.c_void_p(stream))
                    _lib.check(rc)
                try:
                    row[f"dbg{dbg}"] = round(1000 * time_fn(run, reps=10), 1)
                except Exception as e:  # noqa: BLE001
                    row[f"dbg{dbg}"] = str(e)[:60]
            os.environ["PPB_GEMM_DBG"] = "0"
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
