"""Achieved HBM bandwidth of the elementwise / reduction kernels of the step
(north_star: 'achieved HBM GB/s for the elementwise and activation kernels'),
from an ncu --metrics capture (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of one bench step.  ncu replays each kernel with cold
caches and serialised, so this is the per-launch DRAM traffic and rate.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:'pool_fwd|conv_merge|dense_conv|splitk_epilogue|colsum|bias_update|loss_head|im2col|reduce_mask' \
        --clock-control none --csv --log-file ew.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline
    python tools/ew_ncu.py ew.csv [hbm_peak_gbs]
"""
import csv
import json
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6547.8
    hdr = None
    per = defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", ""))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        if d["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(unit, 1e-9)
        elif d["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[key][d["Metric Name"]] = v
    agg = defaultdict(lambda: {"launches": 0, "s": 0.0, "bytes": 0.0})
    for (_, name), m in per.items():
        a = agg[name]
        a["launches"] += 1
        a["s"] += m.get("gpu__time_duration.sum", 0.0)
        a["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["s"]):
        gbs = a["bytes"] / a["s"] / 1e9 if a["s"] > 0 else 0.0
        print(json.dumps({"kernel": name, "launches": a["launches"], "us_total": a["s"] * 1e6,
                          "dram_MB_total": a["bytes"] / 1e6, "achieved_GBs": gbs, "frac_of_hbm": gbs / peak}))


if __name__ == "__main__":
    main()
