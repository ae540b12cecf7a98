"""Float64 PyTorch-CPU restatement of the partitioned step for nets with
conv layers (TEST INFRASTRUCTURE).

The reference has no convolution ("parity unpinned by the
reference"), so this follows the reference's semantics on the conv
extension: forward per micro-batch, loss and gradients in the sum
convention accumulated over micro-batches in order, update
W -= alpha * (acc / b), alpha *= 1 - decay (train_partitioned.cpp:504-512,
632-651).  Partitioning only reorders the dgrad sums, so the
unpartitioned fp64 model is the reference.  Layouts: images NHWC, conv
weights [C_out][k][k][C_in], a dense layer after a conv reads the pooled
output flattened in (c, h, w) order.
"""
import numpy as np
import torch
import torch.nn.functional as Fn


def split_microbatches(b, m):
    sizes = [b // m] * m
    for k in range(b % m):
        sizes[k] += 1
    return sizes


def _forward(layers, params, x):
    a = x
    for lay, (w, b) in zip(layers, params):
        if lay.conv is not None:
            c = lay.conv
            cin = lay.in_units()
            wt = w.reshape(w.shape[0], c.ksize, c.ksize, cin).permute(0, 3, 1, 2)
            if a.dim() == 2:
                a = a.reshape(a.shape[0], c.height, c.width, cin).permute(0, 3, 1, 2)
            a = Fn.conv2d(a, wt, b, padding=c.pad)
            if int(lay.act) == 1:
                a = torch.relu(a)
            if c.pool == 2:
                a = Fn.max_pool2d(a, 2)
        else:
            if a.dim() == 4:
                a = a.reshape(a.shape[0], -1)  # (c, h, w) flatten
            a = a @ w.t() + b
            if int(lay.act) == 1:
                a = torch.relu(a)
    return a


def train(net, X, y, alpha0, decay, iterations, m=1):
    """Returns (W_packed, b_packed, loss_hist, acc_hist) with CE + softmax head."""
    layers = net.layers
    params = [(torch.tensor(l.weights, dtype=torch.float64, requires_grad=True),
               torch.tensor(l.bias, dtype=torch.float64, requires_grad=True)) for l in layers]
    Xt = torch.tensor(np.asarray(X, np.float64))
    if layers[0].conv is not None:
        c = layers[0].conv
        Xt = Xt.reshape(-1, c.height, c.width, layers[0].in_units()).permute(0, 3, 1, 2)
    yt = torch.tensor(np.asarray(y, np.int64))
    b = Xt.shape[0]
    alpha = alpha0
    lh, ah = [], []
    for _ in range(iterations):
        acc = [(torch.zeros_like(w), torch.zeros_like(bb)) for w, bb in params]
        tot, correct, off = 0.0, 0, 0
        for mb in split_microbatches(b, m):
            xb, yb = Xt[off:off + mb], yt[off:off + mb]
            q = _forward(layers, params, xb)
            logp = torch.log_softmax(q, dim=1)
            loss = -logp[torch.arange(mb), yb].clamp(max=690.7755278982137).sum()
            grads = torch.autograd.grad(loss, [t for pair in params for t in pair])
            for i in range(len(params)):
                acc[i] = (acc[i][0] + grads[2 * i], acc[i][1] + grads[2 * i + 1])
            tot += loss.item()
            correct += int((q.argmax(dim=1) == yb).sum())
            off += mb
        with torch.no_grad():
            for (w, bb), (gw, gb) in zip(params, acc):
                w -= alpha * (gw / b)
                bb -= alpha * (gb / b)
        alpha *= 1.0 - decay
        lh.append(tot / b)
        ah.append(correct / b)
    W = np.concatenate([w.detach().numpy().ravel() for w, _ in params])
    B = np.concatenate([bb.detach().numpy().ravel() for _, bb in params])
    return W, B, np.array(lh), np.array(ah)


def forward_acts(net, X):
    """Per-layer outputs (post activation / pool), conv outputs in NHWC."""
    layers = net.layers
    params = [(torch.tensor(l.weights), torch.tensor(l.bias)) for l in layers]
    a = torch.tensor(np.asarray(X, np.float64))
    if layers[0].conv is not None:
        c = layers[0].conv
        a = a.reshape(-1, c.height, c.width, layers[0].in_units()).permute(0, 3, 1, 2)
    outs = []
    for i in range(len(layers)):
        a = _forward(layers[i:i + 1], params[i:i + 1], a)
        outs.append(a.permute(0, 2, 3, 1).reshape(a.shape[0], -1).numpy() if a.dim() == 4 else a.numpy())
    return outs
