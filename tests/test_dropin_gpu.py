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
