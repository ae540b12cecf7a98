"""fwd vs dgrad vs wgrad of one conv layer shape through ppb_debug_conv, with
the epilogue-store probe (PPB_GEMM_DBG=2).  Diagnostic only."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11019_b200 import _lib  # noqa: E402


def run(which, N, H, W, Cin, u, dbg="0", reps=20, bn=0):
    os.environ["PPB_GEMM_DBG"] = dbg
    os.environ["PPB_HALO_DBG"] = dbg
    r4 = lambda x: (x + 3) // 4 * 4
    x_pad = torch.randn(N, H + 2, W + 2, r4(Cin), device="cuda")
    w = torch.randn(u, 9, (Cin + 31) // 32 * 32, device="cuda")
    d_pad = torch.randn(N, H + 2, W + 2, r4(u), device="cuda")
    rows = N * H * W
    if which in (2, 3):
        out = torch.zeros(u, 9 * ((Cin + 31) // 32 * 32), device="cuda")
    else:
        out = torch.empty(rows, r4(u if which == 0 else Cin), device="cuda")
    lib = _lib.lib()

    def call():
        rc = lib.ppb_debug_conv(which, C.c_void_p(x_pad.data_ptr()), N, H, W, Cin, r4(Cin), 1, 3,
                                C.c_void_p(w.data_ptr()), u, C.c_void_p(d_pad.data_ptr()), r4(u),
                                C.c_void_p(out.data_ptr()), out.shape[1], bn, None)
        _lib.check(rc)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * rows * u * 9 * Cin
    print(f"which={which} N={N} {H}x{W} C={Cin} u={u} dbg={dbg} bn={bn}: {ms*1000:.1f} us {fl/ms/1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wgrad":
        for shp in ((512, 8, 8, 128, 256), (512, 4, 4, 256, 512), (512, 8, 8, 256, 256), (512, 4, 4, 512, 512),
                    (512, 16, 16, 128, 128), (512, 16, 16, 64, 128)):
            for which in (2, 3):
                run(which, *shp)
        sys.exit(0)
    for shp in ((512, 8, 8, 256, 256), (512, 4, 4, 512, 512), (512, 2, 2, 512, 512), (512, 8, 8, 128, 256)):
        for which in (0, 1, 3):
            for dbg in ("0", "2"):
                run(which, *shp, dbg=dbg)
