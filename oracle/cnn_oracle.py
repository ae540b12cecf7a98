"""Float64 PyTorch-CPU restatement of the partitioned step, for nets with conv
layers and for dense nets too large for the scalar C oracle (TEST
INFRASTRUCTURE: only tests/, smoke() and bench.py's CPU-baseline legs use it).

The reference has no convolution, so for conv layers this
follows the reference's semantics on the conv extension.  The dense
semantics are the reference's own and are PINNED to it: tests/test_oracle.py
(`test_cnn_oracle_pinned_*`) runs every golden `verify_instances` entry and
the MLP 784-512-512-10 configuration of tests/golden/reference_golden.json
(generated from the compiled, unmodified reference) through `train`, once
with dense layers and once with every dense layer restated as a 1x1 conv over
a 1x1 grid (the conv code path of this module), and requires agreement with
the reference's weights and loss / accuracy histories to 1e-12.

Semantics followed (file:line in /root/reference/proj/src):
  * forward q = a_prev W^T + b, act relu / identity / softmax_last
    (tinynet.cpp:198-213, 96-117);
  * loss: cross entropy -log(max(p_label, 1e-300)) on a softmax head, MSE
    0.5 (out - t)^2 with one-hot targets, or the label value for a 1-wide
    output (tinynet.cpp:120-133, 216-241); loss_history = sum_j loss_sum_j / b
    (train_partitioned.cpp:671,678);
  * gradients in the sum convention, accumulated over micro-batches j = 1..m
    in order (train_partitioned.cpp:504-512), ReLU mask q <= 0 => 0
    (tinynet.cpp:89-94, 252; torch's relu'(0) = 0 matches);
  * update W -= alpha * (acc / b), alpha *= 1 - decay (train_partitioned.cpp:632-651);
  * accuracy: predict_classes (1-wide: out >= 0.5; else the first argmax) and
    the binary-label accuracy() (tinynet.cpp:354-380), or multiclass
    pred == label when `binary_acc=False` (the GPU's multiclass_accuracy).
Partitioning only reorders the dgrad sums, so the
unpartitioned fp64 model is the reference for every plan.  Layouts: images
NHWC, conv weights [C_out][k][k][C_in], a dense layer after a conv reads the
pooled output flattened in (c, h, w) order.
"""
import numpy as np
import torch
import torch.nn.functional as Fn

RELU, IDENTITY, SOFTMAX = 1, 0, 2
MSE, CE = 0, 1


def split_microbatches(b, m):
    """schedule.cpp:46-55: sizes floor(b/m) / ceil(b/m), larger first."""
    sizes = [b // m] * m
    for k in range(b % m):
        sizes[k] += 1
    return sizes


def _shortcut(src, like):
    """ResNet shortcut of a residual layer (the residual extension of the
    conv layer description, include/pipeplan_b200.h ppb_layer.res_from):
    identity, or "option A" (He et al. 2016, §4.2) -- every f-th position of
    the source, its channels zero-padded to the layer's width."""
    f = src.shape[2] // like.shape[2]
    s = src[:, :, ::f, ::f] if f > 1 else src
    if s.shape[1] < like.shape[1]:
        s = torch.cat([s, s.new_zeros(s.shape[0], like.shape[1] - s.shape[1], s.shape[2], s.shape[3])], dim=1)
    return s


def _forward(layers, params, x, flatten=True, outs=None):
    """outs: per-layer outputs so far (residual sources); layers index from len(outs)."""
    a = x
    outs = [] if outs is None else outs
    for lay, (w, b) in zip(layers, params):
        if lay.conv is not None:
            c = lay.conv
            cin = lay.in_units()
            wt = w.reshape(w.shape[0], c.ksize, c.ksize, cin).permute(0, 3, 1, 2)
            if a.dim() == 2:
                a = a.reshape(a.shape[0], c.height, c.width, cin).permute(0, 3, 1, 2)
            a = Fn.conv2d(a, wt, b, padding=c.pad, stride=getattr(c, "stride", 1))
            if getattr(c, "res_from", 0):
                a = a + _shortcut(outs[c.res_from - 1], a)
            if int(lay.act) == RELU:
                a = torch.relu(a)
            if getattr(c, "pool_avg", False) and c.pool > 1:
                a = Fn.avg_pool2d(a, c.pool)
            elif c.pool == 2:
                a = Fn.max_pool2d(a, 2)
        else:
            if a.dim() == 4:
                a = a.reshape(a.shape[0], -1)  # (c, h, w) flatten
            a = a @ w.t() + b
            if int(lay.act) == RELU:
                a = torch.relu(a)
        outs.append(a)
    if flatten and a.dim() == 4:
        a = a.reshape(a.shape[0], -1)
    return a


def _head(q, last_act):
    if last_act == SOFTMAX:
        return torch.softmax(q, dim=1)
    return q  # relu already applied by _forward; identity


def _loss_sum(out, yb, loss, last_act):
    """tinynet.cpp:216-241 (sum over the micro-batch rows)."""
    if loss == CE:
        if last_act != SOFTMAX:
            raise RuntimeError("cross_entropy needs probability outputs (softmax last layer required)")
        p = out[torch.arange(out.shape[0]), yb]
        return -torch.log(torch.clamp(p, min=1e-300)).sum()
    if last_act == SOFTMAX:
        raise RuntimeError("softmax output requires the cross_entropy loss")
    if out.shape[1] == 1:
        t = yb.to(torch.float64).reshape(-1, 1)
    else:
        t = Fn.one_hot(yb, out.shape[1]).to(torch.float64)
    return 0.5 * ((out - t) ** 2).sum()


def predict_classes(out):
    """tinynet.cpp:354-368."""
    if out.shape[1] == 1:
        return (out[:, 0] >= 0.5).to(torch.int64)
    return out.argmax(dim=1)  # first maximum on ties


def _accuracy(pred, y, binary):
    """tinynet.cpp:370-380 (binary) or multiclass pred == label."""
    if binary and not bool(((y == 0) | (y == 1)).all()):
        raise ValueError("accuracy expects binary labels")
    return float((pred == y).sum()) / len(y)


def train(net, X, y, alpha0, decay, iterations, m=1, loss=CE, binary_acc=False):
    """Returns (W_packed, b_packed, loss_hist, acc_hist)."""
    layers = net.layers
    last_act = int(layers[-1].act)
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
    flat = [t for pair in params for t in pair]
    for it in range(iterations):
        acc = [torch.zeros_like(t) for t in flat]
        tot, off = 0.0, 0
        preds = []
        for mb in split_microbatches(b, m):
            xb, yb = Xt[off:off + mb], yt[off:off + mb]
            out = _head(_forward(layers, params, xb), last_act)
            ls = _loss_sum(out, yb, loss, last_act)
            grads = torch.autograd.grad(ls, flat)
            acc = [a + g for a, g in zip(acc, grads)]  # micro-batch order j = 1..m
            tot += ls.item()
            preds.append(predict_classes(out.detach()))
            off += mb
        lv = tot / b
        if not np.isfinite(lv):
            raise RuntimeError(f"diverged at iteration {it + 1}")
        with torch.no_grad():
            for t, g in zip(flat, acc):
                t -= alpha * (g / b)
        alpha *= 1.0 - decay
        lh.append(lv)
        ah.append(_accuracy(torch.cat(preds), yt, binary_acc))
    W = np.concatenate([w.detach().numpy().ravel() for w, _ in params])
    B = np.concatenate([bb.detach().numpy().ravel() for _, bb in params])
    return W, B, np.array(lh), np.array(ah)


def train_layers(net, X, y, alpha0, decay, iterations, m=1, loss=CE):
    """Like train(), but returns the trained per-layer (W, b) list (for per-layer comparisons)."""
    W, B, lh, ah = train(net, X, y, alpha0, decay, iterations, m, loss)
    out, wo, bo = [], 0, 0
    for l in net.layers:
        out.append((W[wo:wo + l.weights.size].reshape(l.weights.shape), B[bo:bo + l.bias.size]))
        wo += l.weights.size
        bo += l.bias.size
    return out, lh, ah


def forward_acts(net, X):
    """Per-layer outputs (post activation / pool), conv outputs in NHWC."""
    layers = net.layers
    params = [(torch.tensor(l.weights), torch.tensor(l.bias)) for l in layers]
    a = torch.tensor(np.asarray(X, np.float64))
    if layers[0].conv is not None:
        c = layers[0].conv
        a = a.reshape(-1, c.height, c.width, layers[0].in_units()).permute(0, 3, 1, 2)
    outs, raw = [], []
    for i in range(len(layers)):
        a = _forward(layers[i:i + 1], params[i:i + 1], a, flatten=False, outs=raw)
        outs.append(a.permute(0, 2, 3, 1).reshape(a.shape[0], -1).numpy() if a.dim() == 4 else a.numpy())
    return outs


# ---------------------------------------------------------------- TF32 arithmetic model

def tf32(t, mode="trunc"):
    """Operand as the tcgen05 kind::tf32 MMA sees it: the fp32 value with the
    low 13 mantissa bits dropped (`trunc`) or rounded to nearest (`rne`)."""
    u = t.to(torch.float32).contiguous().view(torch.int32)
    if mode == "rne":
        u = u + 0x1000
    u = u & ~0x1FFF
    return u.view(torch.float32).to(torch.float64)


def _f32(t):
    return t.to(torch.float32).to(torch.float64)


def train_model(net, X, y, alpha0, decay, iterations, m=1, tf32_mode=None):
    """The partitioned step with an EXPLICIT backward (no autograd), as the GPU
    evaluates it: every GEMM / conv operand rounded as `tf32(mode)` when
    `tf32_mode` is set, products accumulated in float64, activations / error
    signals / parameters stored as float32, bias gradients summed from the
    stored error signal.  With tf32_mode=None and fp32 rounding disabled this
    is the same math as train() (tests/test_oracle.py pins the two against each
    other to 1e-12); with tf32_mode set it is the arithmetic model of the
    GPU's TF32 path, used to separate "the kernels compute what they should"
    (tight) from "TF32 vs the fp64 reference" (looser, stated).  CE + softmax
    head, multiclass accuracy.  Returns (W, b, loss_hist)."""
    if any(l.conv is not None and (getattr(l.conv, "res_from", 0) or getattr(l.conv, "pool_avg", False) or
                                   getattr(l.conv, "stride", 1) > 1) for l in net.layers):
        raise NotImplementedError("train_model: residual / average-pool / strided layers (use train, autograd)")
    exact = tf32_mode is None
    T = (lambda t: t) if exact else (lambda t: tf32(t, tf32_mode))
    S = (lambda t: t) if exact else _f32
    layers = net.layers
    P = [[S(torch.tensor(l.weights, dtype=torch.float64)), S(torch.tensor(l.bias, dtype=torch.float64))]
         for l in layers]
    Xt = torch.tensor(np.asarray(X, np.float64))
    c0 = layers[0].conv
    if c0 is not None:
        Xt = Xt.reshape(-1, c0.height, c0.width, layers[0].in_units()).permute(0, 3, 1, 2)
    Xt = S(Xt)
    yt = torch.tensor(np.asarray(y, np.int64))
    b = Xt.shape[0]
    alpha = alpha0
    lh = []
    for _ in range(iterations):
        acc = [[torch.zeros_like(w), torch.zeros_like(bb)] for w, bb in P]
        tot, off = 0.0, 0
        for mb in split_microbatches(b, m):
            xb, yb = Xt[off:off + mb], yt[off:off + mb]
            ins, qs, idxs, shapes = [], [], [], []
            a = xb
            for lay, (w, bb) in zip(layers, P):
                if lay.conv is not None:
                    c = lay.conv
                    if a.dim() == 2:
                        a = a.reshape(a.shape[0], c.height, c.width, lay.in_units()).permute(0, 3, 1, 2)
                    w4 = w.reshape(w.shape[0], c.ksize, c.ksize, lay.in_units()).permute(0, 3, 1, 2)
                    ins.append(a)
                    q = S(Fn.conv2d(T(a), T(w4), None, padding=c.pad) + bb.reshape(1, -1, 1, 1))
                else:
                    if a.dim() == 4:
                        a = a.reshape(a.shape[0], -1)
                    ins.append(a)
                    q = S(T(a) @ T(w).t() + bb)
                qs.append(q)
                r = torch.relu(q) if int(lay.act) == RELU else q
                if lay.conv is not None and lay.conv.pool == 2:
                    shapes.append(r.shape)
                    r, ix = Fn.max_pool2d(r, 2, return_indices=True)
                    idxs.append(ix)
                else:
                    shapes.append(None)
                    idxs.append(None)
                a = r
            q = qs[-1]
            p = torch.softmax(q, dim=1)
            tot += float(-torch.log(torch.clamp(p[torch.arange(mb), yb], min=1e-300)).sum())
            d = p.clone()
            d[torch.arange(mb), yb] -= 1.0
            d = S(d)
            for li in range(len(layers) - 1, -1, -1):
                lay, (w, bb), xin = layers[li], P[li], ins[li]
                if lay.conv is not None:
                    c = lay.conv
                    w4 = w.reshape(w.shape[0], c.ksize, c.ksize, lay.in_units()).permute(0, 3, 1, 2)
                    gw = torch.nn.grad.conv2d_weight(T(xin), w4.shape, T(d), padding=c.pad)
                    acc[li][0] += gw.permute(0, 2, 3, 1).reshape(w.shape)
                    acc[li][1] += d.sum(dim=(0, 2, 3))
                    if li > 0:
                        d = torch.nn.grad.conv2d_input(xin.shape, T(w4), T(d), padding=c.pad)
                else:
                    acc[li][0] += T(d).t() @ T(xin)
                    acc[li][1] += d.sum(dim=0)
                    if li > 0:
                        d = T(d) @ T(w)
                if li > 0:
                    below = layers[li - 1]
                    if below.conv is not None:
                        pooled = idxs[li - 1] is not None
                        hq, wq = (qs[li - 1].shape[2] // 2, qs[li - 1].shape[3] // 2) if pooled else qs[li - 1].shape[2:]
                        d = d.reshape(d.shape[0], below.fan_out(), hq, wq)
                        if pooled:
                            d = Fn.max_unpool2d(d, idxs[li - 1], 2, output_size=shapes[li - 1][2:])
                    if int(below.act) == RELU:
                        d = d * (qs[li - 1] > 0)
                    d = S(d)
            off += mb
        lh.append(tot / b)
        for (w, bb), (gw, gb) in zip(P, acc):
            w -= alpha * (gw / b)
            bb -= alpha * (gb / b)
            w.copy_(S(w))
            bb.copy_(S(bb))
        alpha *= 1.0 - decay
    W = np.concatenate([w.numpy().ravel() for w, _ in P])
    B = np.concatenate([bb.numpy().ravel() for _, bb in P])
    return W, B, np.array(lh)
