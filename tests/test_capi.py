"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/pipeplan_b200.h declares (no compute call without a GPU)."""
import os
import re

import pytest

from paper_2207_11019_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "pipeplan_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ppb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.EXPORTED), set(names) - set(_lib.EXPORTED)
    assert not L.missing_symbols


def test_library_is_sm100a_tcgen05():
    """The shipped library carries tcgen05 / TMA SASS for sm_100a."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        import pytest

        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out
    assert "UTMALDG" in out
    assert "LDTM" in out


def test_version_and_error_slot():
    L = _lib.lib()
    assert b"sm_100a" in L.ppb_version()
    assert L.ppb_last_error() is not None


def test_cli_usage_errors_exit_2(tmp_path):
    """pipeplan_b200 (dropin/cli_main.cpp): usage errors exit 2 without touching
    a GPU; `plan` is pure host code (serialize_plan)."""
    import json
    import subprocess

    exe = os.path.join(ROOT, "dropin", "_build", "pipeplan_b200")
    if not os.path.exists(exe):
        pytest.skip("dropin/_build/pipeplan_b200 not built (needs the reference sources)")
    for args in (["demo", "-n", "0"], ["frobnicate"], [], ["demo", "--update", "maybe"], ["plan", "--dims", "5"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and "usage error" in r.stderr, (args, r.stderr)
    r = subprocess.run([exe, "plan", "--dims", "8,6,4", "-n", "2", "-Z", "2", "--out", str(tmp_path)],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    doc = json.loads((tmp_path / "plan.json").read_text())
    assert doc["n"] == 2 and len(doc["submodules"]) == 2 and len(doc["boundaries"]) == 1
