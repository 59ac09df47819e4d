"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
K = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # which kernel section
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = rows[starts[K]:starts[K + 1]]
print(sec[0][1][:120])
hdr = sec[1]
data = [dict(zip(hdr, r)) for r in sec[2:] if len(r) == len(hdr)]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
agg = {s: sum(int(d[s] or 0) for d in data) for s in stalls}
print(sorted(agg.items(), key=lambda x: -x[1])[:8])
idx = {d["Address"]: i for i, d in enumerate(data)}
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:n]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((k, int(d[k] or 0)) for k in stalls), key=lambda x: -x[1])[:2]
    print(f"{idx[d['Address']]:5d} {s:6d} {100*s/tot:5.1f}% {d['Instructions Executed']:>8} {d['Source'][:60]:60s} {top}")
