"""Time the GEMM epilogue variants on epilogue-heavy shapes (diagnostic)."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11019_b200 import _lib  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import time_fn  # noqa: E402


def main():
    L = _lib.lib()
    stream = torch.cuda.current_stream().cuda_stream
    for (M, N, K, mode, a_mn, b_mn) in [(524288, 64, 28, 0, 0, 0), (524288, 64, 576, 0, 0, 0), (131072, 128, 1152, 0, 0, 0),
                                        (4096, 8192, 8192, 0, 0, 0), (8192, 8192, 4096, 2, 1, 1), (4096, 8192, 8192, 0, 0, 1)]:
        A = torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, (K + 3) // 4 * 4, device="cuda")
        B = torch.randn(K, N, device="cuda") if b_mn else torch.randn(N, (K + 3) // 4 * 4, device="cuda")
        Cc = torch.zeros(M, N, device="cuda")
        bias = torch.randn(N, device="cuda")
        alpha = torch.tensor([1e-3], device="cuda", dtype=torch.float64)
        flag = torch.zeros(1, device="cuda", dtype=torch.int32)

        def run():
            rc = L.ppb_debug_gemm(C.c_void_p(A.data_ptr()), A.shape[0], K if not a_mn else M, A.shape[1], a_mn,
                                  C.c_void_p(B.data_ptr()), B.shape[0], K if not b_mn else N, B.shape[1], b_mn,
                                  M, N, K, mode, C.c_void_p(Cc.data_ptr()), N, C.c_void_p(bias.data_ptr()), 1, None, 0,
                                  C.c_void_p(alpha.data_ptr()), 1.0, C.c_void_p(flag.data_ptr()), 0, 0,
                                  C.c_void_p(stream))
            _lib.check(rc)
        ms = time_fn(run, reps=10)
        print(json.dumps({"M": M, "N": N, "K": K, "mode": mode, "rowwise": os.environ.get("PPB_EPI_ROWWISE", "0"),
                          "ms": ms, "tflops": 2.0 * M * N * K / ms / 1e9,
                          "out_GBs": M * N * 4 * (2 if mode == 2 else 1) / ms / 1e6}))


if __name__ == "__main__":
    if len(sys.argv) == 1:
        for v in ("0", "1"):
            subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, PPB_EPI_ROWWISE=v), check=False)
    else:
        main()
