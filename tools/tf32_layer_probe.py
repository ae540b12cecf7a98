"""Per-layer activations / error signals of the GPU wide-MLP step against the
TF32 arithmetic model (truncated operands) and fp64 (diagnostic)."""
import os
import sys

sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np
import torch

import bench
import cnn_oracle
from paper_2207_11019_b200 import api
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode

torch.set_num_threads(os.cpu_count())
net, X, y = bench.synthetic_batch("wide_mlp", 1)
ctx = api.Context([0])
s = api.Session(ctx, net, X.shape[0], api.build_plan(net, 1, 1), 1, UpdateMode.async_per_module,
                TrainConfig(alpha0=0.0, decay=0.0, iterations=1), PartitionedTrainOptions(multiclass_accuracy=True))
s.load_batch(X, y)
s.step(1)
s.sync()
f32 = lambda t: t.to(torch.float32).to(torch.float64)
for mode in (None, "trunc"):
    T = (lambda t: t) if mode is None else (lambda t: cnn_oracle.tf32(t, mode))
    a = f32(torch.tensor(X, dtype=torch.float64))
    acts, qs = [], []
    for l in net.layers:
        W = f32(torch.tensor(l.weights)); b = f32(torch.tensor(l.bias))
        q = f32(T(a) @ T(W).t() + b)
        qs.append(q)
        a = torch.relu(q) if int(l.act) == 1 else q
        acts.append(a)
    p = torch.softmax(qs[-1], 1)
    d = p.clone(); d[torch.arange(len(y)), torch.tensor(y, dtype=torch.long)] -= 1
    ds = [None] * 4
    ds[3] = f32(d)
    for li in (3, 2, 1):
        W = f32(torch.tensor(net.layers[li].weights))
        d = f32((T(ds[li]) @ T(W)) * (qs[li - 1] > 0))
        ds[li - 1] = d
    for l in (1, 2, 3):
        g = s.read_tensor(0, l)
        r = acts[l - 1].numpy()
        print(mode, "a", l, "rel", np.linalg.norm(g - r) / np.linalg.norm(r), "maskdiff", np.mean((g > 0) != (r > 0)), flush=True)
    for l in (1, 2, 3, 4):
        g = s.read_tensor(2, l)
        r = ds[l - 1].numpy()
        print(mode, "delta", l, "rel", np.linalg.norm(g - r) / np.linalg.norm(r), flush=True)
