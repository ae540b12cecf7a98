"""bench.py end to end on the GPU: the default VGG-16 line (driver contract
keys), and the multi-device step at full batch with every plan device on
cuda:0 (the N > 1 path of the driver's scaling run, on one GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_vgg16_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert 0 < d["roofline"]["frac"] < 1.5 and d["roofline"]["bound"] == "tensor"
    assert d["config"]["workload"] == "vgg16" and d["config"]["batch"] == 512


def test_bench_vgg16_multi_device_plan_on_one_gpu():
    """Same data, seeds and step count: the 2- and 4-device plans reach the
    1-device loss (TF32 tolerance; shards only reorder the dgrad sums)."""
    ref = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"])["loss_last"]
    assert 0.5 < ref < 5.0
    for k in (2, 4):
        d = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"], env={"PPB_BENCH_PLAN_DEVICES": str(k)})
        assert d["value"] > 0
        assert abs(d["loss_last"] - ref) <= 2e-3 * ref, (k, d["loss_last"], ref)
