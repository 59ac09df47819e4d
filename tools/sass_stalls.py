"""Top SASS lines by warp-stall samples from `ncu -i X --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
stall_cols = [h for h in hdr if h.startswith("stall_")]
top = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for d in top[:n]:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    reasons = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{c}={v:.0f}" for v, c in reasons if v > 0)
    print(f"{100 * s / tot:5.1f}% {d['Address']:>6} {d['Source'][:60]:60s} {rs}")
