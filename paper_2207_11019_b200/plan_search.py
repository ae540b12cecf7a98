"""Plan chooser for the B200 executor.

The reference chooses plans with `optimize_plan` (proj/src/cost.cpp:151-238):
candidates are span cuts x merge masks over `build_plan_with_cuts`, priced by
`task_costs` (cost.cpp:25-69) as per-sample FLOPs / a nominal device rate plus
an alpha-beta link term for sub-module boundaries only; staged device groups
come from `build_staged_plan` (partition.cpp:123-138).  That model cannot tell
a B200 plan that scales from one that does not: it charges nothing for the
per-layer all-gather / reduce-scatter inside a sub-module, nothing for narrow
shards running at a fraction of the tensor-core rate, and it sums task times
instead of simulating the pipelined schedule.

Here:

* **Calibration** (`calibrate`): the per-shard device time of every layer is
  MEASURED on the B200 through the product itself -- a `Session` on the plan
  `build_plan(net, g, 1)` with g logical plan devices on one GPU and m
  micro-batches, one serialised eager step with CUDA events around every op
  (`Session.profile_ops`) -- for shard groups g in {1, 2, 4, 8} and
  micro-batch counts m in {1, 2, 4, 8}.  Per layer it keeps the forward
  (shard GEMM + pool / loss head) and input-gradient (dgrad + merge) time per
  shard per micro-batch, and the weight-gradient + SGD time per shard per
  step (the executor runs wgrad once over all b rows).  The ratio of the
  CUDA-graph step to the serialised sum at g = m = 1 (the graph overlaps the
  wgrad stream with the forward / dgrad chain) is kept as `overlap`.
* **Links**: NVLink 5 through NVSwitch, alpha-beta: beta = 770 GB/s per
  direction per GPU, the peer-copy bandwidth measured on this pool
  (B200_PROFILING.md, "NVLink"), alpha = 5 us.  One GPU is available to this
  build, so these are the guide's measured references, not a measurement of
  this run.  Inside a stage the merges are fused into the producing epilogue
  (DESIGN §5), so a layer costs max(compute, all-gather) forward and
  max(compute, reduce-scatter) backward; a stage boundary costs a gather at
  the hub plus a broadcast (the executor's concat path).
* **Candidates**: every stage count Z <= min(n, L), contiguous layer spans x
  device-group sizes (compositions of n, from the calibrated widths) found by
  dynamic programming on the bottleneck stage, plus the reference's
  all-layers-over-n plans (`build_plan(g, n, Z)`), each at every calibrated m.
* **Pricing**: an event simulation of the executor's schedule (one resource
  per stage group; F(s, j) after F(s-1, j) and, with the pipeline gate of
  schedule.cpp:293-296, after B(s, j-2); B(s, j) after B(s+1, j); ready ops
  by smaller j, then B before F, as the reference's priority rule
  schedule.cpp:185-203; the stage's wgrad + SGD once after its last B), the
  makespan scaled by the measured `overlap`.

`choose_plan` returns the cheapest plan with its predicted step time and the
predicted speed-up over the best one-GPU plan; `bench.py --gpus N` runs the
chosen plan and prints the prediction beside the measurement.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import api
from .api import BoundaryKind, PartitionPlan, SubModule

NVLINK_BW = 770e9   # B/s per direction per GPU (B200_PROFILING.md, peer copy measured on this pool)
NVLINK_ALPHA = 5e-6  # s per transfer

FWD_KINDS = ("fwd_gemm", "pool_relayout", "loss_head")
BWD_KINDS = ("dgrad_gemm", "conv_merge", "bwd_merge")
UPD_KINDS = ("wgrad_sgd_gemm", "bias_update")


@dataclass
class Calibration:
    workload: str
    batch: int
    layers: int
    # key "g,m" -> per layer [fwd_ms per shard per micro-batch, bwd_ms per shard
    # per micro-batch, upd_ms per shard per step]
    table: Dict[str, List[List[float]]] = field(default_factory=dict)
    overlap: float = 1.0
    graph_step_ms: float = 0.0
    out_feats: List[int] = field(default_factory=list)  # per-sample output elements per layer
    in_feats: List[int] = field(default_factory=list)
    source: str = ""

    def gs(self) -> List[int]:
        return sorted({int(k.split(",")[0]) for k in self.table})

    def ms(self) -> List[int]:
        return sorted({int(k.split(",")[1]) for k in self.table})

    def layer_times(self, l: int, g: int, m: int) -> Tuple[float, float, float]:
        """(fwd, bwd, upd) seconds of layer l (1-based) at shard group g, m micro-batches."""
        row = self.table[f"{g},{m}"][l - 1]
        return row[0] * 1e-3, row[1] * 1e-3, row[2] * 1e-3

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            json.dump(self.__dict__, f, indent=1)

    @staticmethod
    def load(path: str) -> "Calibration":
        with open(path) as f:
            return Calibration(**json.load(f))


def _layer_feats(net: api.TinyNet) -> Tuple[List[int], List[int]]:
    outs, ins = [], []
    for l in net.layers:
        c = l.conv
        if c is None:
            ins.append(l.fan_in())
            outs.append(l.fan_out())
        else:
            ins.append(c.height * c.width * l.in_units())
            h, w = c.out_hw()
            q = 2 if c.pool == 2 else 1
            outs.append((h // q) * (w // q) * l.fan_out())
    return outs, ins


def calibrate(workload: str, net: api.TinyNet, X, y, gs: Sequence[int] = (1, 2, 4, 8),
              ms: Sequence[int] = (1, 2, 4, 8)) -> Calibration:
    """Per-layer shard times measured on the B200 (one GPU, g logical devices)."""
    from .api import PartitionedTrainOptions, TrainConfig, UpdateMode

    batch = X.shape[0]
    L = len(net.layers)
    outs, ins = _layer_feats(net)
    cal = Calibration(workload, batch, L, out_feats=outs, in_feats=ins,
                      source="Session.profile_ops on one B200 (g logical plan devices on cuda:0), "
                             "CUDA events around every op of one serialised eager step")
    for g in gs:
        if min(net.dims()[1:]) < g:
            continue
        for m in ms:
            if batch // m < 1:
                continue
            plan = api.build_plan(net, g, 1)
            s = api.Session(api.Context([0] * g), net, batch, plan, m, UpdateMode.async_per_module,
                            TrainConfig(alpha0=1e-4, decay=1e-2, iterations=1),
                            PartitionedTrainOptions(multiclass_accuracy=True, use_graph=True, pipeline_gate=2))
            s.load_batch(X, y)
            s.step(2)
            s.sync()
            if g == 1 and m == 1:
                cal.graph_step_ms = s.time_steps(20) / 20
            s.profile(1)
            ops = s.profile_ops()
            rows = [[0.0, 0.0, 0.0] for _ in range(L)]
            for o in ops:
                l = o["layer"]
                if not 1 <= l <= L:
                    continue
                if o["kind"] in FWD_KINDS:
                    rows[l - 1][0] += o["ms"] / (g * m)
                elif o["kind"] in BWD_KINDS:
                    rows[l - 1][1] += o["ms"] / (g * m)
                elif o["kind"] in UPD_KINDS:
                    rows[l - 1][2] += o["ms"] / g
            cal.table[f"{g},{m}"] = rows
            if g == 1 and m == 1:
                serial = sum(o["ms"] for o in ops)
                cal.overlap = cal.graph_step_ms / serial if serial > 0 else 1.0
            del s
    return cal


# ------------------------------------------------------------------ plans


def plan_from_spans(net, cuts: Sequence[int], groups: Sequence[Sequence[int]], n: int) -> PartitionPlan:
    """partition.cpp:80-107 (plan_from_spans): sub-module j owns layers
    (cuts[j-1], cuts[j]] on devices groups[j]; shards from split_layer."""
    g = api.model_graph_of(net) if isinstance(net, api.TinyNet) else net
    L = g.num_layers()
    subs, first = [], 1
    for j, devs in enumerate(groups):
        last = cuts[j] if j < len(groups) - 1 else L
        shards = [api.split_layer(g.layers[l - 1], list(devs)) for l in range(first, last + 1)]
        subs.append(SubModule(j + 1, first, last, list(devs), shards))
        first = last + 1
    return PartitionPlan(n, subs, [BoundaryKind.concat_repartition] * (len(groups) - 1))


@dataclass
class Stage:
    first: int
    last: int
    g: int


def _stage_costs(cal: Calibration, st: Stage, m: int, rows: int, link_bw: float, alpha: float):
    """(F, B, U) seconds of one stage: per micro-batch forward and backward
    (compute vs fused all-gather / reduce-scatter), per step wgrad + SGD."""
    F = B = U = 0.0
    for l in range(st.first, st.last + 1):
        f, b, u = cal.layer_times(l, st.g, m)
        if st.g > 1:
            ag = alpha + (st.g - 1) / st.g * rows * cal.out_feats[l - 1] * 4 / link_bw
            rs = alpha + (st.g - 1) / st.g * rows * cal.in_feats[l - 1] * 4 / link_bw if l > 1 else 0.0
            f, b = max(f, ag), max(b, rs)
        F += f
        B += b
        U += u
    return F, B, U


def simulate(cal: Calibration, stages: Sequence[Stage], m: int, gate: int = 2, link_bw: float = NVLINK_BW,
             alpha: float = NVLINK_ALPHA) -> float:
    """Makespan (s) of one step of the executor's schedule for a staged plan."""
    Z = len(stages)
    rows = cal.batch / m
    costs = [_stage_costs(cal, s, m, rows, link_bw, alpha) for s in stages]
    # boundary s -> s+1: gather at the hub + broadcast to the next group
    bnd = []
    for s in range(Z - 1):
        by = rows * cal.out_feats[stages[s].last - 1] * 4
        bnd.append(2 * alpha + by / link_bw + (by / link_bw if stages[s + 1].g > 1 else 0.0))
    done: Dict[Tuple[str, int, int], float] = {}
    free = [0.0] * Z
    pending = {(k, s, j) for s in range(Z) for j in range(m) for k in ("F", "B")}

    def ready_time(op):
        k, s, j = op
        deps = []
        if k == "F":
            if s > 0:
                deps.append(("F", s - 1, j, bnd[s - 1]))
            if j - gate >= 0:
                deps.append(("B", s, j - gate, 0.0))
        else:
            deps.append(("F", s, j, 0.0))
            if s < Z - 1:
                deps.append(("B", s + 1, j, bnd[s]))
        t = 0.0
        for dk, ds, dj, lag in deps:
            key = (dk, ds, dj)
            if key not in done:
                return None
            t = max(t, done[key] + lag)
        return t

    while pending:
        best = None
        for op in pending:
            r = ready_time(op)
            if r is None:
                continue
            k, s, j = op
            start = max(r, free[s])
            # earliest start, then smaller j, then B before F (schedule.cpp:185-203)
            key = (start, j, 0 if k == "B" else 1, s)
            if best is None or key < best[0]:
                best = (key, op)
        (start, _, _, s), op = best
        k, _, j = op
        dur = costs[s][0] if k == "F" else costs[s][1]
        done[op] = start + dur
        free[s] = start + dur
        pending.discard(op)
    # wgrad + SGD of each stage once its micro-batches' backward is done
    end = 0.0
    for s in range(Z):
        end = max(end, max(free[s], max(done[("B", s, j)] for j in range(m))) + costs[s][2])
    return end * cal.overlap


@dataclass
class Choice:
    n: int
    m: int
    stages: List[Stage]
    predicted_s: float
    plan: PartitionPlan
    label: str

    def describe(self) -> dict:
        return {"n": self.n, "m": self.m, "Z": len(self.stages),
                "stages": [{"layers": [s.first, s.last], "gpus": s.g} for s in self.stages],
                "predicted_step_ms": self.predicted_s * 1e3, "label": self.label}


def _compositions_dp(cal: Calibration, n: int, Z: int, m: int, sizes: Sequence[int], link_bw: float,
                     alpha: float, keep: int = 4):
    """Contiguous spans x group sizes (sum n) minimising the bottleneck stage
    m*(F+B)+U; returns up to `keep` stage lists (distinct bottlenecks)."""
    L = cal.layers
    rows = cal.batch / m
    # best[i][d][k] = list of (bottleneck, stages) using layers 1..i, d devices, k stages
    from functools import lru_cache

    @lru_cache(maxsize=None)
    def cost(first, last, g):
        F, B, U = _stage_costs(cal, Stage(first, last, g), m, rows, link_bw, alpha)
        return m * (F + B) + U

    @lru_cache(maxsize=None)
    def solve(i, d, k):
        if k == 0:
            return ((0.0, ()),) if i == 0 and d == 0 else ()
        out = []
        for first in range(k, i + 1):  # stage k covers layers first..i
            for g in sizes:
                if g > d:
                    continue
                c = cost(first, i, g)
                for bott, st in solve(first - 1, d - g, k - 1):
                    out.append((max(bott, c), st + ((first, i, g),)))
        out.sort()
        return tuple(out[:keep])

    return [[Stage(*t) for t in st] for _, st in solve(L, n, Z)]


def choose_plan(net, n: int, cal: Calibration, ms: Optional[Sequence[int]] = None, link_bw: float = NVLINK_BW,
                alpha: float = NVLINK_ALPHA) -> Tuple[Choice, List[Choice]]:
    """Cheapest predicted plan for n GPUs (and every candidate priced)."""
    L = cal.layers
    sizes = [g for g in cal.gs() if g <= n]
    ms = [m for m in (ms or cal.ms()) if f"1,{m}" in cal.table]
    cands: List[Choice] = []
    for m in ms:
        if f"{n},{m}" in cal.table:  # the reference's build_plan(g, n, 1): every layer over all n
            st = [Stage(1, L, n)]
            cands.append(Choice(n, m, st, simulate(cal, st, m, link_bw=link_bw, alpha=alpha), None,
                                "build_plan(n, Z=1)"))
        for Z in range(2, min(n, L) + 1):
            for st in _compositions_dp(cal, n, Z, m, [g for g in sizes if f"{g},{m}" in cal.table], link_bw, alpha):
                cands.append(Choice(n, m, st, simulate(cal, st, m, link_bw=link_bw, alpha=alpha), None,
                                    f"staged Z={Z}"))
    cands.sort(key=lambda c: (c.predicted_s, len(c.stages), c.m))
    best = cands[0]
    dev, groups = 1, []
    for s in best.stages:
        groups.append(list(range(dev, dev + s.g)))
        dev += s.g
    best.plan = plan_from_spans(net, [s.last for s in best.stages[:-1]], groups, n)
    return best, cands


def predicted_scaling(net, cal: Calibration, ns: Sequence[int] = (1, 2, 4, 8)) -> dict:
    base, _ = choose_plan(net, 1, cal)
    out = {}
    for n in ns:
        if n > max(cal.gs()) and n != 1:
            continue
        c, _ = choose_plan(net, n, cal)
        sp = base.predicted_s / c.predicted_s
        out[str(n)] = {**c.describe(), "predicted_speedup": sp, "predicted_frac_of_linear": sp / n}
    return out


def default_calibration_path(workload: str) -> str:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return os.path.join(root, "profiles", f"calib_{workload}.json")
