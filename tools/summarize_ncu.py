"""Summarise an ncu launch list (--metrics gpu__time_duration.sum) and a
--set full capture into profiles/.

    python tools/summarize_ncu.py <tag> <workload>
reads gpurun_out/<tag>_launches.csv and gpurun_out/<tag>_gemm.ncu-rep.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second", "l1tex__m_xbar2l1tex_read_bytes.sum",
            "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct"]
    res = []
    for r in rows[2:]:
        res.append({w: (r[hdr.index(w)] + " " + units[hdr.index(w)]).strip() for w in want if w in hdr})
    return res


def to_bytes(s):
    v, u = s.split()[0].replace(",", ""), s.split()[1]
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main():
    tag, workload = sys.argv[1], sys.argv[2]
    rep = sys.argv[3] if len(sys.argv) > 3 else "gemm"  # gpurun_out/<tag>_<rep>.ncu-rep
    out_name = f"{tag}_ncu.md" if rep == "gemm" else f"{tag}_{rep}_ncu.md"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary {tag} ({workload})", ""]
    lpath = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
    if os.path.exists(lpath) and rep == "gemm":
        agg = launches(lpath)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, "
               "cold-cache, serialised: compare shares)", "",
               "| kernel | launches | total ns | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| `{k}` | {n} | {t:.0f} | {t / tot:.1%} |")
        md.append("")
    fpath = os.path.join(ROOT, "gpurun_out", f"{tag}_{rep}.ncu-rep")
    if os.path.exists(fpath):
        res = full(fpath)
        md += ["## `--set full` capture of the dominant kernel", ""]
        for i, r in enumerate(res):
            md.append(f"### launch {i}")
            for k, v in r.items():
                md.append(f"- {k}: {v}")
            md.append("")
        tr = [to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"]) for r in res]
        tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
        d = json.load(open(tpath)) if os.path.exists(tpath) else {}
        d[workload] = sum(tr) / len(tr)
        d[f"{workload}_source"] = f"profiles/{out_name} (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
        json.dump(d, open(tpath, "w"), indent=1)
    open(os.path.join(ROOT, "profiles", out_name), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
