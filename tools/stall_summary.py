"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples by reason and the hottest SASS instructions (with neighbours)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    col = {h: i for i, h in enumerate(hdr)}
    samp = col["Warp Stall Sampling (All Samples)"]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[samp] or 0) for r in body)
    print(f"{path}: {len(body)} SASS lines, {tot:.0f} samples")
    agg = {h: sum(float(r[col[h]] or 0) for r in body) for h in reasons}
    for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {h:28s} {v:8.0f}  {100 * v / max(tot, 1):5.1f}%")
    idx = sorted(range(len(body)), key=lambda i: -float(body[i][samp] or 0))[:top]
    for i in sorted(idx):
        r = body[i]
        why = sorted(((float(r[col[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
        print(f"  {i:5d} {float(r[samp]):7.0f} ex={r[col['Instructions Executed']]:>8s} {r[1].strip()[:70]:70s} "
              + " ".join(f"{h}={v:.0f}" for v, h in why if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
