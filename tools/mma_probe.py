"""Drive tools/mma_probe.cu: kind::tf32 MMA rate, A from smem (SS) vs TMEM (TS)
vs TS with a tcgen05.cp of A per K-block, at N = 64 / 128 / 256.
Prints one JSON line per case (TFLOP/s over 148 SMs at the measured clock)."""
import ctypes as C
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    lib = C.CDLL(os.path.join(HERE, "_mma_probe.so"))
    lib.mma_probe.argtypes = [C.c_int] * 5 + [C.c_void_p, C.c_void_p]
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    kb, iters = 4, 2000
    for n in (64, 128, 256):
        for mode in (0, 1, 2):
            for rep in range(2):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                rc = lib.mma_probe(n, mode, kb, iters, ctas, C.c_void_p(cyc.data_ptr()), None)
                e.record()
                torch.cuda.synchronize()
                if rc != 0:
                    print(json.dumps({"n": n, "mode": mode, "error": rc}))
                    sys.exit(1)
            ms = s.elapsed_time(e)
            flop = 2.0 * 128 * n * 32 * kb * iters * ctas
            c = cyc.double().mean().item()
            print(json.dumps({"n": n, "mode": ["SS", "TS", "TS+cp"][mode], "ms": ms, "tflops": flop / ms / 1e9,
                              "cycles_per_kblock": c / (kb * iters),
                              "macs_per_clk_per_sm": 128 * n * 32 / (c / (kb * iters))}))


if __name__ == "__main__":
    main()
