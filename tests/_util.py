"""Shared test helpers (fixtures, oracle loading, distances)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.json")
sys.path.insert(0, os.path.join(ROOT, "oracle"))

_golden = None


def golden():
    global _golden
    if _golden is None:
        with open(GOLDEN) as f:
            _golden = json.load(f)
    return _golden


def oracle():
    from oracle import Oracle  # noqa: E402  (test infrastructure)

    return Oracle()


def reference_or_none():
    from oracle import REF_SO, Reference

    return Reference() if os.path.exists(REF_SO) else None


def net_distance(W1, b1, W2, b2):
    """verify.cpp:64-81: max |x-y| / max(1, |x|, |y|) over all parameters."""
    x = np.concatenate([np.ravel(W1), np.ravel(b1)])
    y = np.concatenate([np.ravel(W2), np.ravel(b2)])
    return float(np.max(np.abs(x - y) / np.maximum(1.0, np.maximum(np.abs(x), np.abs(y))))) if x.size else 0.0


def rel_norm(x, ref):
    ref = np.asarray(ref, np.float64)
    d = np.linalg.norm(np.asarray(x, np.float64) - ref)
    n = np.linalg.norm(ref)
    return float(d / n) if n > 0 else float(d)
