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
        for mode in (0, 1, 2, 3, 4):
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
            print(json.dumps({"n": n, "mode": ["SS", "TS", "TS+cp", "SS-2acc", "SS-4acc"][mode], "ms": ms, "tflops": flop / ms / 1e9,
                              "cycles_per_kblock": c / (kb * iters),
                              "macs_per_clk_per_sm": 128 * n * 32 / (c / (kb * iters))}))


def main2():
    """probe2: the product kernel's issue structure (elect_one around 4
    back-to-back MMAs per K-block) with 1 / 2 / 4 round-robin accumulators."""
    lib = C.CDLL(os.path.join(HERE, "_mma_probe.so"))
    lib.mma_probe2.argtypes = [C.c_int] * 5 + [C.c_void_p]
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    kb, iters = 4, 2000
    for n, nacc in ((64, 1), (64, 2), (64, 4), (128, 1), (128, 2), (128, 4), (256, 1), (256, 2)):
        for rep in range(2):
            rc = lib.mma_probe2(n, nacc, kb, iters, ctas, C.c_void_p(cyc.data_ptr()))
            torch.cuda.synchronize()
            if rc != 0:
                print(json.dumps({"n": n, "nacc": nacc, "error": rc}))
                continue
            c = cyc.double().mean().item()
            if rep == 1:
                print(json.dumps({"probe": "kernel-issue", "n": n, "nacc": nacc,
                                  "cycles_per_mma": c / (kb * iters * 4),
                                  "macs_per_clk_per_sm": 128 * n * 32 / (c / (kb * iters)),
                                  "frac_of_2048": 128 * n * 32 / (c / (kb * iters)) / 2048}))


def main3():
    """probe3: descriptors as base + constant steps, GROUP k-blocks (4 x GROUP
    back-to-back MMAs) per elect region."""
    lib = C.CDLL(os.path.join(HERE, "_mma_probe.so"))
    lib.mma_probe3.argtypes = [C.c_int] * 5 + [C.c_void_p]
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    kb, iters = 4, 2000
    for n, grp in ((64, 1), (64, 2), (64, 4), (128, 1), (128, 2), (128, 4), (256, 1)):
        for rep in range(2):
            rc = lib.mma_probe3(n, grp, kb, iters, ctas, C.c_void_p(cyc.data_ptr()))
            torch.cuda.synchronize()
            c = cyc.double().mean().item()
            if rc == 0 and rep == 1:
                print(json.dumps({"probe": "cheap-issue", "n": n, "kblocks_per_issue": grp,
                                  "cycles_per_mma": c / (kb * iters * 4),
                                  "frac_of_2048": 128 * n * 32 / (c / (kb * iters)) / 2048}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "3":
        main3()
    elif len(sys.argv) > 1 and sys.argv[1] == "2":
        main2()
    else:
        main()
