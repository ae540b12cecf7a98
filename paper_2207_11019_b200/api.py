"""Python mirror of the reference `pipeplan` API for the partitioned step.

Names, argument meaning and error behaviour follow the reference C++ headers
(include/pipeplan/{tinynet,partition,schedule,train_partitioned}.hpp) so the
tests read like the reference's own.  Everything below is a thin layer over
the C ABI (include/pipeplan_b200.h): planning runs in the native planner,
training on the GPU kernels.  There is no host/CPU fallback.

Exceptions: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::runtime_error -> PipeplanError (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import PipeplanError, check

__all__ = [
    "ActKind", "LossKind", "UpdateMode", "BoundaryKind", "LayerSpec", "ModelGraph", "Shard", "SubModule",
    "PartitionPlan", "ConvSpec", "TinyLayer", "TinyNet", "Batch", "TrainConfig", "PartitionedTrainOptions", "TrainResult",
    "split_layer", "split_microbatches", "build_plan", "build_staged_plan", "build_plan_with_cuts",
    "merge_submodules", "merge_all", "validate_plan", "serialize_plan", "parse_plan", "model_graph_of", "train_partitioned", "Context",
    "Session", "PipeplanError",
]

_i = C.POINTER(C.c_int)
_d = C.POINTER(C.c_double)
_f = C.POINTER(C.c_float)


def _ip(a):
    return a.ctypes.data_as(_i)


def _dp(a):
    return a.ctypes.data_as(_d)


class ActKind(IntEnum):  # tinynet.hpp:38
    identity = 0
    relu = 1
    softmax_last = 2


class LossKind(IntEnum):  # tinynet.hpp:39
    mse = 0
    cross_entropy = 1


class UpdateMode(IntEnum):  # schedule.hpp:12
    none = 0
    sync_barrier = 1
    async_per_module = 2


class BoundaryKind(IntEnum):  # partition.hpp:36
    concat_repartition = 0
    direct = 1


@dataclass
class LayerSpec:  # model.hpp:12-21 (dense chain subset)
    id: int
    fan_in: int
    fan_out: int
    fwd_flops: float = 0.0


@dataclass
class ModelGraph:  # model.hpp:23-29
    layers: List[LayerSpec]
    name: str = "chain"

    def num_layers(self) -> int:
        return len(self.layers)


@dataclass
class Shard:  # partition.hpp:14-24
    layer_id: int
    device_id: int
    lo: int
    hi: int
    replicated: bool = False

    def units(self) -> int:
        return self.hi - self.lo


@dataclass
class SubModule:  # partition.hpp:26-38
    index: int
    first_layer: int
    last_layer: int
    devices: List[int]
    shards: List[List[Shard]]

    def num_layers(self) -> int:
        return self.last_layer - self.first_layer + 1

    def layer_shards(self, layer_id: int) -> List[Shard]:
        return self.shards[layer_id - self.first_layer]


@dataclass
class PartitionPlan:  # partition.hpp:40-47
    n: int
    submodules: List[SubModule]
    boundaries: List[BoundaryKind]
    provenance: List[str] = field(default_factory=list)

    def num_submodules(self) -> int:
        return len(self.submodules)

    # flat encoding of include/pipeplan_b200.h
    def to_flat(self) -> np.ndarray:
        f = [self.n, len(self.submodules)]
        for sm in self.submodules:
            f += [sm.index, sm.first_layer, sm.last_layer, len(sm.devices), *sm.devices]
            for row in sm.shards:
                for s in row:
                    f += [s.layer_id, s.device_id, s.lo, s.hi, int(s.replicated)]
        f += [int(b) for b in self.boundaries]
        return np.asarray(f, np.int32)

    @staticmethod
    def from_flat(flat, provenance=None) -> "PartitionPlan":
        f = [int(x) for x in flat]
        r = 0

        def nxt():
            nonlocal r
            r += 1
            return f[r - 1]

        n, Z = nxt(), nxt()
        subs = []
        for _ in range(Z):
            idx, first, last, D = nxt(), nxt(), nxt(), nxt()
            devs = [nxt() for _ in range(D)]
            shards = []
            for _l in range(first, last + 1):
                shards.append([Shard(nxt(), nxt(), nxt(), nxt(), bool(nxt())) for _d in range(D)])
            subs.append(SubModule(idx, first, last, devs, shards))
        bounds = [BoundaryKind(nxt()) for _ in range(Z - 1)]
        return PartitionPlan(n, subs, bounds, list(provenance or []))


@dataclass
class ConvSpec:
    """Convolution extension of a layer (BASELINE CNN configs; the reference is
    dense-only): stride-1 ksize x ksize conv with zero padding over an input of
    height x width x C_in (NHWC), then an optional 2x2 max pool (pool = 2)."""
    height: int
    width: int
    ksize: int = 3
    pad: int = 1
    pool: int = 1
    # residual extension (ResNet-style configs): add the output of layer
    # `res_from` (1-based, 0 = none) to the pre-activation -- identity, or
    # every f-th position with zero-padded channels ("option A") -- and pool
    # with a pool x pool average instead of the 2x2 max (`pool_avg`)
    res_from: int = 0
    pool_avg: bool = False
    stride: int = 1

    def conv_hw(self):
        """Conv output grid before pooling."""
        return ((self.height + 2 * self.pad - self.ksize) // self.stride + 1,
                (self.width + 2 * self.pad - self.ksize) // self.stride + 1)

    def out_hw(self):
        ho = (self.height + 2 * self.pad - self.ksize) // self.stride + 1
        wo = (self.width + 2 * self.pad - self.ksize) // self.stride + 1
        return ho // self.pool, wo // self.pool


@dataclass
class TinyLayer:  # tinynet.hpp:41-48
    weights: np.ndarray  # fan_out x fan_in (dense) | C_out x (ksize*ksize*C_in) (conv), float64
    bias: np.ndarray     # fan_out | C_out
    act: ActKind = ActKind.identity
    conv: Optional[ConvSpec] = None

    def fan_in(self) -> int:
        return self.weights.shape[1]

    def fan_out(self) -> int:
        return self.weights.shape[0]

    def in_units(self) -> int:
        return self.weights.shape[1] // (self.conv.ksize ** 2) if self.conv else self.weights.shape[1]

    def out_features(self) -> int:
        if self.conv is None:
            return self.fan_out()
        h, w = self.conv.out_hw()
        return self.fan_out() * h * w

    def fwd_flops(self) -> float:
        if self.conv is None:
            return 0.0  # default_costs (model.cpp:124-137) applies
        c = self.conv
        ho, wo = c.conv_hw()
        return 2.0 * self.weights.shape[0] * self.weights.shape[1] * ho * wo

    def to_c(self) -> _lib.LayerC:
        lc = _lib.LayerC()
        lc.kind = 1 if self.conv else 0
        lc.in_units, lc.out_units, lc.act = self.in_units(), self.fan_out(), int(self.act)
        if self.conv:
            lc.height, lc.width, lc.ksize, lc.pad, lc.pool = (self.conv.height, self.conv.width, self.conv.ksize,
                                                              self.conv.pad, self.conv.pool)
            lc.res_from, lc.pool_kind, lc.stride = self.conv.res_from, int(self.conv.pool_avg), self.conv.stride
        return lc


@dataclass
class TinyNet:  # tinynet.hpp:50-56
    layers: List[TinyLayer]

    def num_layers(self) -> int:
        return len(self.layers)

    def has_conv(self) -> bool:
        return any(l.conv is not None for l in self.layers)

    def layers_c(self):
        arr = (_lib.LayerC * len(self.layers))()
        for i, l in enumerate(self.layers):
            arr[i] = l.to_c()
        return arr

    def dims(self) -> List[int]:
        return [self.layers[0].fan_in()] + [l.fan_out() for l in self.layers]

    def acts(self) -> List[int]:
        return [int(l.act) for l in self.layers]

    def pack(self):
        W = np.concatenate([np.ascontiguousarray(l.weights, np.float64).ravel() for l in self.layers])
        b = np.concatenate([np.ascontiguousarray(l.bias, np.float64).ravel() for l in self.layers])
        return W, b

    @staticmethod
    def unpack(dims, acts, W, b) -> "TinyNet":
        layers, wo, bo = [], 0, 0
        for l in range(len(acts)):
            fi, fo = dims[l], dims[l + 1]
            layers.append(TinyLayer(W[wo: wo + fi * fo].reshape(fo, fi).copy(), b[bo: bo + fo].copy(), ActKind(acts[l])))
            wo += fi * fo
            bo += fo
        return TinyNet(layers)

    def replace_params(self, W, b) -> "TinyNet":
        """Same architecture, parameters from packed arrays (pack() layout)."""
        layers, wo, bo = [], 0, 0
        for l in self.layers:
            n = l.weights.size
            layers.append(TinyLayer(W[wo: wo + n].reshape(l.weights.shape).copy(), b[bo: bo + l.bias.size].copy(),
                                    l.act, l.conv))
            wo += n
            bo += l.bias.size
        return TinyNet(layers)


@dataclass
class Batch:  # tinynet.hpp:58-63
    X: np.ndarray       # b x input_dim
    labels: np.ndarray  # b

    def size(self) -> int:
        return self.X.shape[0]


@dataclass
class TrainConfig:  # tinynet.hpp:76-82
    alpha0: float = 1e-4
    decay: float = 1e-2
    loss: LossKind = LossKind.cross_entropy
    iterations: int = 50
    seed: int = 1


@dataclass
class PartitionedTrainOptions:  # train_partitioned.hpp:9-11 + GPU knobs
    receive_timeout_s: float = 30.0
    precision: str = "tf32"          # "tf32" (tcgen05) | "fp32" (CUDA-core FMA chains)
    multiclass_accuracy: bool = False
    use_graph: bool = True
    pipeline_gate: int = 2
    # activation stash policy (simulate.hpp:14-16 MemoryMode): "stash_all" is
    # the reference executor (every micro-batch resident, weight gradients over
    # all b rows); "proposed" keeps min(m, pipeline_gate) micro-batches and
    # accumulates weight gradients per micro-batch
    memory_mode: str = "stash_all"
    # merge transport of dense layers inside a sub-module: "p2p" (fused
    # epilogue peer stores) or "nccl" (ncclAllGather / ncclReduceScatter;
    # one plan device per GPU)
    merge_backend: str = "p2p"

    def to_c(self) -> _lib.OptionsC:
        o = _lib.OptionsC()
        o.receive_timeout_s = self.receive_timeout_s
        o.precision = {"tf32": 0, "fp32": 1}[self.precision]
        o.multiclass_accuracy = int(self.multiclass_accuracy)
        o.use_graph = int(self.use_graph)
        o.pipeline_gate = int(self.pipeline_gate)
        o.memory_mode = {"stash_all": 0, "proposed": 1}[self.memory_mode]
        o.merge_backend = {"p2p": 0, "nccl": 1}[self.merge_backend]
        return o


@dataclass
class TrainResult:  # tinynet.hpp:110-114
    net: TinyNet
    loss_history: List[float]
    acc_history: List[float]


# ---------------------------------------------------------------- planner

def _chain(g):
    if isinstance(g, TinyNet):
        g = model_graph_of(g)
    if isinstance(g, ModelGraph):
        fi = np.asarray([l.fan_in for l in g.layers], np.int32)
        fo = np.asarray([l.fan_out for l in g.layers], np.int32)
        fw = np.asarray([l.fwd_flops for l in g.layers], np.float64)
        return fi, fo, fw
    dims = list(g)  # dims list: input then fan_out per layer
    return (np.asarray(dims[:-1], np.int32), np.asarray(dims[1:], np.int32), None)


def model_graph_of(net: TinyNet) -> ModelGraph:
    """tinynet.cpp:463-476 (default costs are applied by the planner).  For
    nets with conv layers the chain is over sharded units (channels) and the
    conv layers carry their FLOPs explicitly."""
    specs, prev = [], None
    conv = net.has_conv()
    for l, layer in enumerate(net.layers):
        fi = layer.in_units() if prev is None else prev
        fl = layer.fwd_flops()
        if conv and layer.conv is None:
            # a dense layer over a flattened conv output: its real fan_in is
            # C*H*W, not the C units the chain shards, so price it explicitly
            fl = 2.0 * layer.fan_in() * layer.fan_out()
        specs.append(LayerSpec(l + 1, fi, layer.fan_out(), fl))
        prev = layer.fan_out()
    return ModelGraph(specs)


def split_layer(layer, devices, replicate_narrow: bool = False) -> List[Shard]:
    """partition.cpp:15-48.  `layer` is a LayerSpec or (layer_id, fan_out);
    `devices` a device list or a count n (devices 1..n)."""
    if isinstance(layer, LayerSpec):
        lid, fo = layer.id, layer.fan_out
    else:
        lid, fo = layer
    devs = list(range(1, devices + 1)) if isinstance(devices, int) else list(devices)
    n = len(devs)
    lo, hi, rep = (np.zeros(max(n, 1), np.int32) for _ in range(3))
    d = np.asarray(devs or [0], np.int32)
    check(_lib.lib().ppb_split_layer(lid, fo, _ip(d), n, int(replicate_narrow), _ip(lo), _ip(hi), _ip(rep)))
    return [Shard(lid, devs[k], int(lo[k]), int(hi[k]), bool(rep[k])) for k in range(n)]


def split_microbatches(b: int, m: int) -> List[int]:
    """schedule.cpp:46-55."""
    out = np.zeros(max(m, 1), np.int32)
    check(_lib.lib().ppb_split_microbatches(b, m, _ip(out)))
    return [int(x) for x in out[:m]]


def _two_call(fn, *args) -> np.ndarray:
    n = C.c_int(0)
    check(fn(*args, None, 0, C.byref(n)))
    out = np.zeros(n.value, np.int32)
    check(fn(*args, _ip(out), n.value, C.byref(n)))
    return out


def build_plan(g, n: int, Z: int, replicate_narrow: bool = False) -> PartitionPlan:
    """partition.cpp:110-121."""
    fi, fo, fw = _chain(g)
    flat = _two_call(_lib.lib().ppb_build_plan, _ip(fi), _ip(fo), _dp(fw) if fw is not None else None,
                     len(fo), n, Z, int(replicate_narrow))
    return PartitionPlan.from_flat(flat)


def build_staged_plan(g, device_groups: Sequence[Sequence[int]], replicate_narrow: bool = False) -> PartitionPlan:
    """partition.cpp:123-138."""
    fi, fo, fw = _chain(g)
    flat_g = np.asarray([d for grp in device_groups for d in grp] or [0], np.int32)
    sizes = np.asarray([len(grp) for grp in device_groups] or [0], np.int32)
    flat = _two_call(_lib.lib().ppb_build_staged_plan, _ip(fi), _ip(fo), _dp(fw) if fw is not None else None,
                     len(fo), _ip(flat_g), _ip(sizes), len(device_groups), int(replicate_narrow))
    return PartitionPlan.from_flat(flat)


def build_plan_with_cuts(g, n: int, cuts: Sequence[int], replicate_narrow: bool = False) -> PartitionPlan:
    """partition.cpp:140-155."""
    fi, fo, _ = _chain(g)
    c = np.asarray(list(cuts) or [0], np.int32)
    flat = _two_call(_lib.lib().ppb_build_plan_with_cuts, _ip(fi), _ip(fo), len(fo), n, _ip(c), len(cuts),
                     int(replicate_narrow))
    return PartitionPlan.from_flat(flat)


def merge_submodules(p: PartitionPlan, group: Sequence[int]) -> PartitionPlan:
    """partition.cpp:157-175."""
    flat = p.to_flat()
    g = np.asarray(list(group) or [0], np.int32)
    check(_lib.lib().ppb_merge_submodules(_ip(flat), len(flat), _ip(g), len(group)))
    prov = list(p.provenance) + [f"merge[{group[0]}..{group[-1]}]"]
    return PartitionPlan.from_flat(flat, prov)


def merge_all(p: PartitionPlan) -> PartitionPlan:
    """partition.cpp:177-182."""
    if p.num_submodules() < 2:
        return p
    return merge_submodules(p, list(range(1, p.num_submodules() + 1)))


def serialize_plan(p: PartitionPlan) -> str:
    """partition.cpp:303-331 (byte-identical JSON)."""
    flat = p.to_flat()
    prov = "\n".join(p.provenance).encode()
    n = C.c_size_t(0)
    L = _lib.lib()
    check(L.ppb_serialize_plan(_ip(flat), len(flat), prov, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(L.ppb_serialize_plan(_ip(flat), len(flat), prov, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def parse_plan(text: str) -> PartitionPlan:
    """partition.cpp:333-384."""
    L = _lib.lib()
    n = C.c_int(0)
    check(L.ppb_parse_plan(text.encode(), None, 0, C.byref(n), None, 0))
    out = np.zeros(n.value, np.int32)
    prov = C.create_string_buffer(len(text) + 1)
    check(L.ppb_parse_plan(text.encode(), _ip(out), n.value, C.byref(n), prov, len(text) + 1))
    p = PartitionPlan.from_flat(out)
    p.provenance = [x for x in prov.value.decode().split("\n") if x] if prov.value else []
    return p


def validate_plan(p: PartitionPlan, g, cluster_devices: int = 0) -> None:
    """partition.cpp:232-294."""
    fi, fo, _ = _chain(g)
    flat = p.to_flat()
    check(_lib.lib().ppb_validate_plan(_ip(flat), len(flat), _ip(fi), _ip(fo), len(fo), cluster_devices))


# ---------------------------------------------------------------- training

class Context:
    """Binds plan devices 1..n to CUDA ordinals (several may share one GPU)."""

    def __init__(self, device_map: Sequence[int]):
        dm = np.asarray(list(device_map), np.int32)
        h = C.c_void_p()
        check(_lib.lib().ppb_context_create(_ip(dm), len(dm), C.byref(h)))
        self._h = h
        self.device_map = list(device_map)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and getattr(_lib, "lib", None) is not None:
            try:
                _lib.lib().ppb_context_destroy(self._h)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self._h = None


def _cfg_c(cfg: TrainConfig) -> _lib.TrainConfigC:
    c = _lib.TrainConfigC()
    c.alpha0, c.decay, c.loss, c.iterations, c.seed = cfg.alpha0, cfg.decay, int(cfg.loss), cfg.iterations, cfg.seed
    return c


class Session:
    """Device-resident partitioned training state (ppb_session_*)."""

    def __init__(self, ctx: Context, net: TinyNet, batch_size: int, plan: PartitionPlan, m: int,
                 mode: UpdateMode, cfg: TrainConfig, opts: Optional[PartitionedTrainOptions] = None):
        opts = opts or PartitionedTrainOptions()
        self._net = net
        self._dims = np.asarray(net.dims(), np.int32)
        self._acts = np.asarray(net.acts(), np.int32)
        W, b = net.pack()
        flat = plan.to_flat()
        h = C.c_void_p()
        self._cfg = _cfg_c(cfg)
        self._opts = opts.to_c()
        if net.has_conv():
            self._layers = net.layers_c()
            check(_lib.lib().ppb_session_create_layers(ctx._h, self._layers, len(net.layers), _dp(W), _dp(b),
                                                       batch_size, _ip(flat), len(flat), m, int(mode),
                                                       C.byref(self._cfg), C.byref(self._opts), C.byref(h)))
        else:
            check(_lib.lib().ppb_session_create(ctx._h, _ip(self._dims), _ip(self._acts), len(self._acts), _dp(W),
                                                _dp(b), batch_size, _ip(flat), len(flat), m, int(mode),
                                                C.byref(self._cfg), C.byref(self._opts), C.byref(h)))
        self._h = h
        self._ctx = ctx
        self.batch_size = batch_size
        self.nW, self.nb = W.size, b.size
        self.in_features = _input_features(net)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and getattr(_lib, "lib", None) is not None:
            try:
                _lib.lib().ppb_session_destroy(self._h)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self._h = None

    def _host_batch(self, X, labels, dtype):
        """The C ABI takes bare pointers: check shapes here (the reference
        throws on a width mismatch in matmul_nt, tinynet.cpp:24-35, and on a
        row / label count mismatch, train_partitioned.cpp:132) and hand it
        contiguous buffers of the exact element types."""
        X = np.asarray(X)
        y = np.ascontiguousarray(labels, np.int32).reshape(-1)
        rows = X.shape[0] if X.ndim else 0
        width = int(np.prod(X.shape[1:])) if X.ndim >= 2 else (0 if X.ndim == 0 else 1)
        if rows != self.batch_size:
            raise ValueError(f"batch has {rows} rows, session was created for {self.batch_size}")
        if y.shape[0] != rows:
            raise ValueError("batch rows and label count disagree")
        if width != self.in_features:
            raise ValueError(f"matmul_nt: inner dimensions disagree (X has {width} columns, "
                             f"the network takes {self.in_features})")
        return np.ascontiguousarray(X.reshape(rows, width), dtype), y

    def load_batch(self, X, labels):
        if np.asarray(X).dtype == np.float32:
            Xc, y = self._host_batch(X, labels, np.float32)
            check(_lib.lib().ppb_session_load_batch_f32(self._h, Xc.ctypes.data_as(_f), _ip(y)))
        else:
            Xc, y = self._host_batch(X, labels, np.float64)
            check(_lib.lib().ppb_session_load_batch(self._h, _dp(Xc), _ip(y)))

    def step(self, iterations: int = 1):
        check(_lib.lib().ppb_session_step(self._h, iterations))

    def sync(self):
        check(_lib.lib().ppb_session_sync(self._h))

    def history(self):
        n = C.c_int(0)
        check(_lib.lib().ppb_session_history(self._h, None, None, 0, C.byref(n)))
        lh = np.zeros(max(n.value, 1))
        ah = np.zeros(max(n.value, 1))
        check(_lib.lib().ppb_session_history(self._h, _dp(lh), _dp(ah), n.value, C.byref(n)))
        return lh[: n.value], ah[: n.value]

    def get_net(self) -> TinyNet:
        W = np.zeros(self.nW)
        b = np.zeros(self.nb)
        check(_lib.lib().ppb_session_get_net(self._h, _dp(W), _dp(b)))
        return self._net.replace_params(W, b)

    def read_tensor(self, kind: int, layer: int, device: int = 1) -> np.ndarray:
        n = C.c_size_t(0)
        check(_lib.lib().ppb_session_read_tensor(self._h, kind, layer, device, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        check(_lib.lib().ppb_session_read_tensor(self._h, kind, layer, device, _dp(out), n.value, C.byref(n)))
        return out.reshape(self.batch_size, -1)

    def time_steps(self, iterations: int) -> float:
        """Device milliseconds of `iterations` steps (CUDA events on the launching stream)."""
        ms = C.c_float(0)
        check(_lib.lib().ppb_session_time_steps(self._h, iterations, C.byref(ms)))
        return ms.value

    OP_KINDS = ("sync", "fwd_gemm", "dgrad_gemm", "wgrad_sgd_gemm", "loss_head", "bwd_merge", "bias_update",
                "finalize", "peer_copy", "pool_relayout", "conv_merge")

    def profile(self, iterations: int = 1) -> dict:
        """Per-op-kind device time / launches / FLOPs over `iterations` eager steps."""
        k = len(self.OP_KINDS)
        ms, cnt, fl = np.zeros(k), np.zeros(k, np.int32), np.zeros(k)
        check(_lib.lib().ppb_session_profile(self._h, iterations, _dp(ms), _ip(cnt), _dp(fl), k))
        return {name: {"ms": float(ms[i]), "launches": int(cnt[i]), "flops": float(fl[i])}
                for i, name in enumerate(self.OP_KINDS) if cnt[i]}

    def profile_ops(self) -> list:
        """Per-op records of the last profile() call."""
        n = C.c_int(0)
        L = _lib.lib()
        check(L.ppb_session_profile_ops(self._h, None, None, None, None, None, 0, C.byref(n)))
        k, lay, inf = (np.zeros(max(n.value, 1), np.int32) for _ in range(3))
        ms, fl = np.zeros(max(n.value, 1)), np.zeros(max(n.value, 1))
        check(L.ppb_session_profile_ops(self._h, _ip(k), _ip(lay), _ip(inf), _dp(ms), _dp(fl), n.value, C.byref(n)))
        return [{"kind": self.OP_KINDS[k[i]] if k[i] < len(self.OP_KINDS) else int(k[i]), "layer": int(lay[i]),
                 "bn": int(inf[i] & 1023), "cg": int((inf[i] >> 10) & 3),
                 "splits": int((inf[i] >> 12) & 4095), "halo": int((inf[i] >> 24) & 1),
                 "ms": float(ms[i]), "tflops": float(fl[i] / ms[i] / 1e9) if ms[i] > 0 else 0.0}
                for i in range(n.value)]

    def profile_concurrent(self, iterations: int = 1) -> None:
        """One eager step with the streams overlapping as in the graph (per-op
        start / end events); read it with profile_timeline() / op_meta()."""
        check(_lib.lib().ppb_session_profile_concurrent(self._h, iterations))

    def op_meta(self) -> list:
        """(micro-batch, plan device, stream role) per op, profile_ops() order
        (the enqueue order of the pipelined schedule)."""
        n = C.c_int(0)
        L = _lib.lib()
        check(L.ppb_session_op_meta(self._h, None, None, None, 0, C.byref(n)))
        mb, dev, role = (np.zeros(max(n.value, 1), np.int32) for _ in range(3))
        check(L.ppb_session_op_meta(self._h, _ip(mb), _ip(dev), _ip(role), n.value, C.byref(n)))
        roles = ("forward", "backward", "wgrad", "main")
        return [{"mb": int(mb[i]), "device": int(dev[i]), "role": roles[role[i]]} for i in range(n.value)]

    def profile_timeline(self) -> list:
        """profile_ops() records with the op's start (ms from the first op) and stream index."""
        ops = self.profile_ops()
        n = C.c_int(0)
        L = _lib.lib()
        st, sid = np.zeros(max(len(ops), 1)), np.zeros(max(len(ops), 1), np.int32)
        check(L.ppb_session_profile_starts(self._h, _dp(st), _ip(sid), len(ops), C.byref(n)))
        for i, o in enumerate(ops):
            o["start"] = float(st[i])
            o["stream"] = int(sid[i])
        return ops

    def step_host(self, X: np.ndarray, labels: np.ndarray) -> float:
        """End-to-end step from host buffers (H2D X/labels, step, D2H loss)."""
        loss = C.c_double(0)
        Xc, y = self._host_batch(X, labels, np.float32)  # no copy when already float32 / int32 contiguous
        check(_lib.lib().ppb_session_step_host(self._h, Xc.ctypes.data_as(_f), _ip(y), C.byref(loss)))
        return loss.value

    def step_host_f64(self, X: np.ndarray, labels: np.ndarray) -> float:
        """step_host with the reference's fp64 batch rows (Batch::X)."""
        loss = C.c_double(0)
        Xc, y = self._host_batch(X, labels, np.float64)
        check(_lib.lib().ppb_session_step_host_f64(self._h, _dp(Xc), _ip(y), C.byref(loss)))
        return loss.value

    def step_host_pipelined(self, X: np.ndarray, labels: np.ndarray) -> float:
        """Streaming step: stages this batch while the previous step runs and
        returns the PREVIOUS step's loss (NaN on the first call)."""
        loss = C.c_double(0)
        if np.asarray(X).dtype == np.float64:
            Xc, y = self._host_batch(X, labels, np.float64)
            check(_lib.lib().ppb_session_step_host_pipelined(self._h, None, _dp(Xc), _ip(y), C.byref(loss)))
        else:
            Xc, y = self._host_batch(X, labels, np.float32)
            check(_lib.lib().ppb_session_step_host_pipelined(self._h, Xc.ctypes.data_as(_f), None, _ip(y),
                                                             C.byref(loss)))
        return loss.value

    def kernels_per_step(self) -> int:
        k = C.c_int(0)
        check(_lib.lib().ppb_session_kernels_per_step(self._h, C.byref(k)))
        return k.value

    def memory(self):
        """(total device bytes, stash bytes): the stash part scales with the
        resident micro-batches (activations, error signals, merge slots)."""
        t, st = C.c_size_t(0), C.c_size_t(0)
        check(_lib.lib().ppb_session_memory(self._h, C.byref(t), C.byref(st)))
        return t.value, st.value


_default_ctx = {}


def _input_features(net: TinyNet) -> int:
    l0 = net.layers[0]
    return l0.in_units() * (l0.conv.height * l0.conv.width if l0.conv else 1)


def device_count() -> int:
    n = C.c_int(0)
    check(_lib.lib().ppb_device_count(C.byref(n)))
    return n.value


def default_device_map(n_dev: int) -> List[int]:
    """Plan device k+1 -> CUDA ordinal k, one plan device per visible GPU; a
    plan with more devices than visible GPUs wraps round-robin (several plan
    devices then share a GPU, which is how multi-device plans run on one)."""
    g = max(1, device_count())
    return [k % g for k in range(n_dev)]


def _context_for(devices):
    key = tuple(devices)
    if key not in _default_ctx:
        _default_ctx[key] = Context(devices)
    return _default_ctx[key]


def train_partitioned(net: TinyNet, batch: Batch, cfg: TrainConfig, plan: PartitionPlan, m: int,
                      mode: UpdateMode, opts: Optional[PartitionedTrainOptions] = None,
                      device_map: Optional[Sequence[int]] = None) -> TrainResult:
    """train_partitioned.cpp:121-709 on B200s.  `device_map[k]` is the CUDA
    ordinal of plan device k+1 (default: default_device_map, one plan device
    per visible GPU)."""
    opts = opts or PartitionedTrainOptions()
    n_dev = max([d for sm in plan.submodules for d in sm.devices] + [plan.n, 1])
    ctx = _context_for(device_map if device_map is not None else default_device_map(n_dev))
    dims = np.asarray(net.dims(), np.int32)
    acts = np.asarray(net.acts(), np.int32)
    W, b = net.pack()
    X = np.ascontiguousarray(batch.X, np.float64)
    y = np.ascontiguousarray(batch.labels, np.int32)
    if X.shape[0] != y.shape[0]:
        raise ValueError("batch rows and label count disagree")
    if int(np.prod(X.shape[1:])) != _input_features(net):
        raise ValueError(f"matmul_nt: inner dimensions disagree (X has {int(np.prod(X.shape[1:]))} columns, "
                         f"the network takes {_input_features(net)})")
    flat = plan.to_flat()
    Wo, bo = np.zeros_like(W), np.zeros_like(b)
    it = max(cfg.iterations, 1)
    lh, ah = np.zeros(it), np.zeros(it)
    cc, oc = _cfg_c(cfg), opts.to_c()
    if net.has_conv():
        X = np.ascontiguousarray(X.reshape(X.shape[0], -1), np.float64)
        check(_lib.lib().ppb_train_partitioned_layers(ctx._h, net.layers_c(), len(net.layers), _dp(W), _dp(b), _dp(X),
                                                      _ip(y), X.shape[0], _ip(flat), len(flat), m, int(mode),
                                                      C.byref(cc), C.byref(oc), _dp(Wo), _dp(bo), _dp(lh), _dp(ah)))
    else:
        check(_lib.lib().ppb_train_partitioned(ctx._h, _ip(dims), _ip(acts), len(acts), _dp(W), _dp(b), _dp(X),
                                               _ip(y), X.shape[0], _ip(flat), len(flat), m, int(mode), C.byref(cc),
                                               C.byref(oc), _dp(Wo), _dp(bo), _dp(lh), _dp(ah)))
    return TrainResult(net.replace_params(Wo, bo), list(lh[: cfg.iterations]), list(ah[: cfg.iterations]))
