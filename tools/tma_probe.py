"""TMA load throughput (bytes per SM clock) vs box shape / swizzle mode,
through ppb_debug_tma_bw (csrc/tma_probe.cu).  The source matrix (64 MB) is
L2-resident after the first pass."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_11019_b200 import _lib  # noqa: E402

L = _lib.lib()
rows, cols = 65536, 256
src = torch.randn(rows, cols, device="cuda")
clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else None


def run(box_rows, mn, boxes, stages, iters=400, ctas=148):
    def call():
        _lib.check(L.ppb_debug_tma_bw(C.c_void_p(src.data_ptr()), rows, cols, box_rows, mn, boxes, stages, iters,
                                      ctas, None))
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byts = ctas * iters * boxes * box_rows * 128
    print(json.dumps({"box_rows": box_rows, "mn_major": mn, "boxes_per_stage": boxes, "stages": stages, "ctas": ctas,
                      "us": round(ms * 1000, 1), "TBps": round(byts / ms / 1e9, 2),
                      "B_per_clk_per_SM_at_1.9GHz": round(byts / (ms * 1e-3) / 1.9e9 / ctas, 1)}), flush=True)


if __name__ == "__main__":
    for mn in (0, 1):
        for box_rows, boxes in ((32, 6), (32, 12), (64, 3), (64, 6), (128, 2), (128, 3), (256, 1), (198, 1)):
            run(box_rows, mn, boxes, 8 if box_rows * boxes * 128 * 8 <= 200000 else 4)
    run(32, 1, 6, 8, ctas=74)
    run(128, 0, 2, 6, ctas=74)
