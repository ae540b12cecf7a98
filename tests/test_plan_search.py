"""Plan chooser (paper_2207_11019_b200/plan_search.py) on CPU: plan
construction is the reference's plan_from_spans (checked against the C-ABI
planner, itself bit-exact to the reference), the simulator reproduces the
closed forms it must, and the chooser returns valid plans over exactly n
devices.  The calibration tables here are synthetic; the measured ones live
in profiles/calib_*.json (tools/calibrate.py on the B200)."""
import numpy as np
import pytest

from paper_2207_11019_b200 import api, configs
from paper_2207_11019_b200.plan_search import (Calibration, Stage, choose_plan, plan_from_spans,
                                               predicted_scaling, simulate)


def _flat(p):
    return p.to_flat().tolist()


def _synthetic(net, batch, gs=(1, 2, 4, 8), ms=(1, 2, 4), fixed_ms=0.01):
    """Shard time = fixed launch cost + FLOPs / (rate x width efficiency)."""
    L = len(net.layers)
    g_model = api.model_graph_of(net)
    cal = Calibration("synthetic", batch, L, overlap=0.85)
    from paper_2207_11019_b200.plan_search import _layer_feats

    cal.out_feats, cal.in_feats = _layer_feats(net)
    for g in gs:
        for m in ms:
            rows = []
            for l, spec in enumerate(g_model.layers):
                fl = spec.fwd_flops or 2.0 * spec.fan_in * spec.fan_out
                u = max(1, spec.fan_out // g)
                eff = min(1.0, u / 256.0) ** 0.5
                t = fl * batch / m / g / (700e12 * eff) * 1e3 + fixed_ms
                rows.append([t, t if l > 0 else 0.0, (t - fixed_ms) * m + fixed_ms])
            cal.table[f"{g},{m}"] = rows
    return cal


def test_plan_from_spans_matches_reference_builders():
    net = configs.mlp784(seed=1)
    for n in (1, 2, 3):
        for cuts in ([], [1], [2], [1, 2]):
            groups = [list(range(1, n + 1))] * (len(cuts) + 1)
            assert _flat(plan_from_spans(net, cuts, groups, n)) == _flat(api.build_plan_with_cuts(net, n, cuts))
    # staged: balanced spans (build_staged_plan) with explicit groups
    groups = [[1, 2], [3]]
    ref = api.build_staged_plan(net, groups)
    cuts = [sm.last_layer for sm in ref.submodules[:-1]]
    assert _flat(plan_from_spans(net, cuts, groups, 3)) == _flat(ref)


def test_simulator_closed_forms():
    net = configs.mlp784(seed=1)
    cal = _synthetic(net, 64)
    L = len(net.layers)
    F = sum(cal.layer_times(l, 1, 1)[0] for l in range(1, L + 1))
    B = sum(cal.layer_times(l, 1, 1)[1] for l in range(1, L + 1))
    U = sum(cal.layer_times(l, 1, 1)[2] for l in range(1, L + 1))
    assert simulate(cal, [Stage(1, L, 1)], 1) == pytest.approx((F + B + U) * cal.overlap)
    # one stage, m micro-batches: the resource is busy throughout
    F2 = sum(cal.layer_times(l, 1, 2)[0] for l in range(1, L + 1))
    B2 = sum(cal.layer_times(l, 1, 2)[1] for l in range(1, L + 1))
    U2 = sum(cal.layer_times(l, 1, 2)[2] for l in range(1, L + 1))
    assert simulate(cal, [Stage(1, L, 1)], 2) == pytest.approx((2 * (F2 + B2) + U2) * cal.overlap)
    # two stages never beat the bottleneck stage's own work, never exceed the serial sum
    st = [Stage(1, 1, 1), Stage(2, L, 1)]
    t = simulate(cal, st, 2) / cal.overlap
    works = []
    for s in st:
        w = 0.0
        for l in range(s.first, s.last + 1):
            f, b, u = cal.layer_times(l, 1, 2)
            w += 2 * (f + b) + u
        works.append(w)
    assert max(works) <= t + 1e-12


@pytest.mark.parametrize("workload,n", [("mlp784", 2), ("mlp784", 4), ("vgg16", 2), ("vgg16", 8), ("wide_mlp", 8)])
def test_choose_plan_valid(workload, n):
    net = {"mlp784": configs.mlp784, "vgg16": configs.vgg16_cifar, "wide_mlp": configs.wide_mlp}[workload](seed=1)
    batch = {"mlp784": 64, "vgg16": 512, "wide_mlp": 4096}[workload]
    cal = _synthetic(net, batch)
    best, cands = choose_plan(net, n, cal)
    api.validate_plan(best.plan, net)
    devs = sorted({d for sm in best.plan.submodules for d in sm.devices})
    assert devs == list(range(1, n + 1))
    assert best.predicted_s == min(c.predicted_s for c in cands)
    assert best.plan.submodules[0].first_layer == 1 and best.plan.submodules[-1].last_layer == len(net.layers)
    sc = predicted_scaling(net, cal, (1, n))
    assert sc["1"]["predicted_speedup"] == pytest.approx(1.0)
    assert np.isfinite(sc[str(n)]["predicted_speedup"])
