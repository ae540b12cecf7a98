"""Second TMA probe: stage depth and CTAs per SM (see tools/tma_probe.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from tma_probe import run  # noqa: E402

run(32, 0, 1, 24)
run(32, 0, 6, 8)
run(128, 0, 1, 8)
run(128, 0, 2, 4)
run(256, 0, 1, 6)
run(32, 0, 6, 4, ctas=296)
run(128, 0, 1, 6, ctas=296)
