"""Drive tools/tma_probe.cu: TMA box throughput, rank-2 vs rank-4 boxes of
16 KB over a [512][34][34][64] fp32 tensor (loads and bulk stores), one CTA
per SM.  Prints GB/s over 148 SMs and bytes/clk/SM."""
import ctypes as C
import json
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    lib = C.CDLL(os.path.join(HERE, "_tma_probe.so"))
    lib.tma_probe.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    t = torch.zeros(512 * 34 * 34 * 64, dtype=torch.float32, device="cuda")
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    iters = 4000
    for mode, name in ((0, "load rank-2"), (1, "load rank-4"), (2, "store rank-2"), (3, "store rank-4")):
        for rep in range(2):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            rc = lib.tma_probe(C.c_void_p(t.data_ptr()), mode, iters, ctas, C.c_void_p(cyc.data_ptr()))
            e.record()
            torch.cuda.synchronize()
            if rc != 0:
                print(json.dumps({"mode": name, "error": rc}))
                break
            if rep == 1:
                ms = s.elapsed_time(e)
                c = cyc.double().mean().item()
                print(json.dumps({"mode": name, "GBs": 16384.0 * iters * ctas / ms / 1e6,
                                  "bytes_per_clk_per_sm": 16384.0 * iters / c}))


if __name__ == "__main__":
    main()
