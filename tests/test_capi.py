"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/pipeplan_b200.h declares (no compute call without a GPU)."""
import os
import re

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
