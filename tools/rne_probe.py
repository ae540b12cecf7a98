import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests")); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
import test_bench_parity_gpu as T
torch.set_num_threads(os.cpu_count())
for wl, a0, st in (("wide_mlp", 1e-2, 1), ("lenet5", 1e-2, 3)):
    net, Wg, bg, lh = T._gpu(wl, 1, a0, st)
    W0, b0 = net.pack()
    W32, b32 = W0.astype(np.float32).astype(np.float64), b0.astype(np.float32).astype(np.float64)
    for mode in ("trunc", "rne"):
        Wm, bm, _ = T._oracle(wl, a0, st, mode)
        print(wl, mode, T._fmt(T._upd(net, Wg, bg, Wm, bm, W32, b32)), flush=True)
