"""The executed schedule against the reference's scheduler / simulator
(SURVEY §8f rank 3): dropin/_build/simulate_b200 runs the reference's
build_schedule (schedule.cpp:207-330, F(i,j) gated on B(i,j-2)),
attach_updates and simulate / memory_compare (simulate.cpp:159-298) compiled
unchanged.  CPU tests pin what the executor mirrors (the pipelined order and
the two-resident-micro-batch bound of the proposed policy); the GPU test
checks the executor's enqueue order against it."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2207_11019_b200 import api
from paper_2207_11019_b200.api import PartitionedTrainOptions, TinyNet, TrainConfig, UpdateMode

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIM = os.path.join(ROOT, "dropin", "_build", "simulate_b200")
DIMS = [64, 96, 80, 40, 10]


def _simulate(tmp_path, plan, m, tf=1.0, tb=2.0):
    if not os.path.exists(SIM):
        pytest.skip("dropin/_build/simulate_b200 not built (needs the reference sources)")
    Z = len(plan.submodules)
    model = {"schema": 1, "name": "t", "layers": [
        {"kind": "dense", "fan_in": DIMS[i], "fan_out": DIMS[i + 1], "param_count": DIMS[i] * DIMS[i + 1],
         "fwd_flops": 1.0, "bwd_flops": 2.0, "act_bytes": 4.0 * DIMS[i + 1]} for i in range(len(DIMS) - 1)]}
    req = {"model": model, "plan": json.loads(api.serialize_plan(plan)), "m": m,
           "tf": [[tf] * m for _ in range(Z)], "tb": [[tb] * m for _ in range(Z)], "samples_per_microbatch": 8}
    p = tmp_path / "req.json"
    p.write_text(json.dumps(req))
    out = subprocess.run([SIM, str(p)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


def _fb(order):
    return ["%s%d.%d" % tuple(t) for t in order if t[0] in ("F", "B")]


def _live_peak(seq, module):
    """Peak resident micro-batches of a module along a device order (F
    allocates, B frees: simulate.cpp:96-110 under MemoryMode::proposed)."""
    live = peak = 0
    for t in seq:
        k, mod = t[0], int(t[1:].split(".")[0])
        if mod != module:
            continue
        live += 1 if k == "F" else -1
        peak = max(peak, live)
    return peak


def _gate_ok(seq, gate=2):
    """F(i, j) comes after B(i, j - gate) (schedule.cpp:293-296)."""
    seen = set()
    for t in seq:
        k, (mod, j) = t[0], map(int, t[1:].split("."))
        if k == "F" and j > gate and ("B%d.%d" % (mod, j - gate)) not in seen:
            return False
        seen.add(t)
    return True


def test_reference_schedule_on_shared_devices(tmp_path):
    """build_plan(n, Z) puts every module on the same devices: the reference's
    work-conserving list schedule runs B(j) as soon as it is ready (ties:
    backward before forward), one micro-batch resident."""
    r = _simulate(tmp_path, api.build_plan(DIMS, 1, 1), 4)
    assert _fb(r["device_order"][0]) == ["F1.1", "B1.1", "F1.2", "B1.2", "F1.3", "B1.3", "F1.4", "B1.4"]
    assert r["peak_live_microbatches"] == [1]
    assert 0.0 < r["memory_ratio"] < 1.0


@pytest.mark.parametrize("groups,m", [([[1, 2], [3, 4]], 4), ([[1], [2], [3], [4]], 6), ([[1], [2, 3]], 8)])
def test_reference_staged_schedule_within_the_executor_ring(tmp_path, groups, m):
    """Staged device groups (build_staged_plan, partition.cpp:123-138): the
    reference's pipelined schedule respects the F(i,j) <- B(i,j-2) gate and
    never holds more than min(m, 2) micro-batches per module -- the ring the
    executor's proposed policy allocates (gate 2)."""
    plan = api.build_staged_plan(DIMS, groups)
    r = _simulate(tmp_path, plan, m)
    assert all(p <= min(m, 2) for p in r["peak_live_microbatches"]), r["peak_live_microbatches"]
    assert max(r["peak_live_microbatches"]) == min(m, 2)
    for lst in r["device_order"]:
        assert _gate_ok(_fb(lst))


@pytest.mark.gpu
@pytest.mark.parametrize("groups,m", [([[1]], 4), ([[1], [2]], 4), ([[1], [2], [3]], 6), ([[1, 2], [3]], 3)])
def test_executor_order_respects_the_reference_gate_and_ring(tmp_path, groups, m):
    """The executor's per-device enqueue order of forward / backward work
    (Session.op_meta) applies the reference's gate (schedule.cpp:293-296) and,
    read as a schedule, keeps at most the ring's min(m, 2) micro-batches of a
    module resident -- the bound the reference's own schedule reaches."""
    rng = np.random.default_rng(0)
    from _util import oracle  # noqa: I001
    W, b = oracle().init_net(DIMS, 3)
    net = TinyNet.unpack(DIMS, [1, 1, 1, 2], W, b)
    plan = api.build_staged_plan(DIMS, groups)
    n = max(d for g in groups for d in g)
    s = api.Session(api.Context([0] * n), net, 48, plan, m, UpdateMode.async_per_module, TrainConfig(iterations=1),
                    PartitionedTrainOptions(memory_mode="proposed"))
    s.load_batch(rng.standard_normal((48, DIMS[0])), np.arange(48) % 2)
    s.step(1)
    s.profile(1)
    ours = {}
    for o, mt in zip(s.profile_ops(), s.op_meta()):
        # B(i, j): input gradients / merges and, under the proposed policy, the
        # micro-batch's weight gradients (a module of only the first layer has
        # no input gradient)
        if mt["mb"] < 0 or mt["device"] == 0 or mt["role"] == "main":
            continue
        mod = next(sm.index for sm in plan.submodules if sm.first_layer <= o["layer"] <= sm.last_layer)
        key = "%s%d.%d" % ("F" if mt["role"] == "forward" else "B", mod, mt["mb"] + 1)
        seq = ours.setdefault(mt["device"], [])
        if key not in seq:
            seq.append(key)
    r = _simulate(tmp_path, plan, m)
    for d, seq in ours.items():
        assert _gate_ok(seq), seq
        for sm in plan.submodules:
            assert _live_peak(seq, sm.index) <= min(m, 2), (d, seq)
    for sm, peak in zip(plan.submodules, r["peak_live_microbatches"]):
        assert peak <= min(m, 2)
