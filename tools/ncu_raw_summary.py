"""One line per kernel launch from `ncu -i X.ncu-rep --page raw --csv`: duration,
SM / DRAM throughput, tensor-pipe activity, DRAM bytes, occupancy, grid, registers.
    python tools/ncu_raw_summary.py X.raw.csv [title]"""
import csv
import sys

COLS = [("dur_us", ["gpu__time_duration.sum"], 1e-3),
        ("sm_pct", ["sm__throughput.avg.pct_of_peak_sustained_elapsed"], 1),
        ("dram_pct", ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                      "dram__throughput.avg.pct_of_peak_sustained_elapsed"], 1),
        ("tensor_pct", ["TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg."
                        "pct_of_peak_sustained_elapsed"], 1),
        ("dram_rd_MB", ["dram__bytes_read.sum"], 1e-6),
        ("dram_wr_MB", ["dram__bytes_write.sum"], 1e-6),
        ("occ_pct", ["sm__warps_active.avg.pct_of_peak_sustained_active"], 1),
        ("grid", ["launch__grid_size"], 1),
        ("regs", ["launch__registers_per_thread"], 1)]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units = rows[0], rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:]]
    unit = dict(zip(hdr, units))
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print(f"{'kernel':62s} " + " ".join(f"{c:>10s}" for c, _, _ in COLS))
    for d in data:
        out = []
        for _, names, scale in COLS:
            v = None
            for n in names:
                if n in d and num(d[n]) is not None:
                    v = num(d[n])
                    u = unit.get(n, "")
                    if n.startswith("gpu__time_duration"):
                        v *= {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3,
                              "ms": 1e6, "msecond": 1e6}.get(u, 1.0)
                    if n.startswith("dram__bytes") and u in ("Kbyte", "KB"):
                        v *= 1e3
                    if n.startswith("dram__bytes") and u in ("Mbyte", "MB"):
                        v *= 1e6
                    if n.startswith("dram__bytes") and u in ("Gbyte", "GB"):
                        v *= 1e9
                    v *= scale
                    break
            out.append(f"{v:10.2f}" if v is not None else f"{'-':>10s}")
        print(f"{d.get('Kernel Name', '')[:62]:62s} " + " ".join(out))


if __name__ == "__main__":
    main()
