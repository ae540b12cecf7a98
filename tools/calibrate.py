"""Measure the plan chooser's calibration table on the B200 and print the
predicted scaling (paper_2207_11019_b200/plan_search.py).

    python tools/calibrate.py vgg16 [out.json]   (default profiles/calib_<workload>.json)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2207_11019_b200 import plan_search  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    out = sys.argv[2] if len(sys.argv) > 2 else plan_search.default_calibration_path(wl)
    net, X, y = bench.synthetic_batch(wl, seed=1)
    gs = (1, 2, 4, 8)
    ms = (1, 2, 4, 8) if wl != "mlp784" else (1, 2)
    cal = plan_search.calibrate(wl, net, X, y, gs=gs, ms=ms)
    cal.save(out)
    sc = plan_search.predicted_scaling(net, cal)
    print(json.dumps({"workload": wl, "calibration": out, "graph_step_ms": cal.graph_step_ms,
                      "overlap": cal.overlap, "predicted_scaling": sc}))


if __name__ == "__main__":
    main()
