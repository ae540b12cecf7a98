"""The reference's own property suite (run_verification, verify.cpp:104-247)
run with pipeplan::train_partitioned replaced by the B200 drop-in
(dropin/train_partitioned_b200.cpp linked into the reference library).

Properties that exercise train_partitioned:
  * mode-equivalence-async-vs-sync (tol 1e-12): exact on the GPU (0.0).
  * oracle-equivalence-sync (tol 1e-6, written for fp64): the GPU computes in
    fp32 / TF32, so we hold it to 2e-5 (fp32) and 5e-3 (tf32) instead.
The other three properties only run the CPU tinynet code and must pass.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "dropin", "_build", "verify_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision,tol", [("fp32", 2e-5), ("tf32", 5e-3)])
def test_reference_verification_suite_on_gpu(precision, tol):
    if not os.path.exists(EXE):
        pytest.skip("dropin/_build/verify_b200 not built (needs the reference sources)")
    env = dict(os.environ, PPB_PRECISION=precision)
    out = subprocess.run([EXE, "100"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr
    rep = {p["name"]: p for p in json.loads(out.stdout)["properties"]}
    print(json.dumps(rep, indent=1))
    assert rep["mode-equivalence-async-vs-sync"]["max_err"] == 0.0
    assert rep["oracle-equivalence-sync"]["max_err"] <= tol
    for name in ("microbatch-invariance", "gradient-correctness", "shard-reassembly"):
        assert rep[name]["pass"], rep[name]


def test_calibrated_optimize_plan_on_gpu(tmp_path):
    """The reference's optimize_plan priced with per-layer seconds measured on
    the B200 (dropin/optimize_main.cpp): a valid plan whose objective is no
    worse than the default build_plan, and a calibrated model document."""
    exe = os.path.join(ROOT, "dropin", "_build", "optimize_b200")
    if not os.path.exists(exe):
        pytest.skip("dropin/_build/optimize_b200 not built (needs the reference sources)")
    model = tmp_path / "model.json"
    out = subprocess.run([exe, "784,512,512,10", "2", "2", "64", str(model)], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr
    last = json.loads(out.stdout.strip().splitlines()[-1])
    assert 0 < last["optimized_objective_s"] <= last["baseline_build_plan_Z1_objective_s"] * (1 + 1e-12)
    assert last["measured_step_fwd_s"] > 0 and last["measured_step_bwd_s"] > 0
    g = json.loads(model.read_text())
    assert len(g["layers"]) == 3 and all(l["fwd_flops"] > 0 and l["bwd_flops"] > 0 for l in g["layers"])


CLI = os.path.join(ROOT, "dropin", "_build", "pipeplan_b200")


def _cli(args, tmp_path, timeout=600):
    if not os.path.exists(CLI):
        pytest.skip("dropin/_build/pipeplan_b200 not built (needs the reference sources)")
    return subprocess.run([CLI, *args, "--out", str(tmp_path)], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("n,Z,update", [(2, 1, "sync"), (3, 2, "async"), (1, 1, "sync")])
def test_cli_demo_paper_defaults(tmp_path, n, Z, update):
    """`pipeplan_b200 demo`: paper §IV.E hyper-parameters
    (batch 6, CE, 50 iterations, alpha 1e-4 decayed 1e-2) on the synthetic
    blobs through the drop-in; history.csv matches the reference's
    train_sequential (the same binary reports it) within the TF32 tolerance."""
    out = _cli(["demo", "--dims", "784,512,512,10", "-n", str(n), "-Z", str(Z), "--update", update], tmp_path)
    assert out.returncode == 0, out.stderr
    rows = (tmp_path / "history.csv").read_text().strip().splitlines()
    assert rows[0] == "iteration,loss,acc" and len(rows) == 51
    plan = json.loads((tmp_path / "plan.json").read_text())
    assert plan["n"] == n and len(plan["submodules"]) == Z
    dist = float(out.stdout.strip().split("net_distance")[-1])
    assert dist <= 5e-3, out.stdout


def test_cli_verify_exit_codes(tmp_path):
    """`pipeplan_b200 verify`: exit 0 when every property passes; the
    injected gradient fault (VerifyOptions::inject_gradient_fault) exits 1 and
    names the failing property."""
    ok = _cli(["verify", "--seeds", "5"], tmp_path)
    assert ok.returncode == 0, ok.stdout + ok.stderr
    rep = json.loads((tmp_path / "verify_report.json").read_text())
    assert all(p["instances"] == 5 for p in rep["properties"] if p["instances"])
    bad = _cli(["verify", "--seeds", "5", "--inject-fault"], tmp_path)
    assert bad.returncode == 1 and "FAILED property" in bad.stderr, bad.stderr
