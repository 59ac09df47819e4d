"""Summarise an ncu CSV launch list with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum (one un-graphed cfg2 update,
tools/profile_ppo.py bf16) into profiles/ncu_traffic.json: per kernel class
launches, serialized time and DRAM bytes per update."""
import collections
import csv
import json
import sys

path, out = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
# long format: one row per (launch, metric)
per = collections.defaultdict(dict)
names = {}
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
for r in rows:
    lid, name, metric, unit, val = r[0], r[4], r[-3], r[-2], r[-1]
    names[lid] = name.split("(")[0].replace("void ", "")
    per[lid][metric] = float(val.replace(",", "")) * scale.get(unit, 1.0)
agg = collections.defaultdict(lambda: dict(launches=0, us=0.0, dram_read=0.0, dram_write=0.0))
for lid, m in per.items():
    k = names[lid]
    k = k[:k.index("<")] if "<" in k else k
    a = agg[k.split("::")[-1]]
    a["launches"] += 1
    a["us"] += m.get("gpu__time_duration.sum", 0.0)
    a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
    a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
tc = agg.get("tc_gemm_kernel", dict(launches=0, us=0.0, dram_read=0.0, dram_write=0.0))
res = {
    "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "--clock-control none python tools/profile_ppo.py bf16 (one cfg2 PPO update, "
              "un-graphed, serialized launches)",
    "tc_gemm_launches_per_update": tc["launches"],
    "tc_gemm_dram_read_bytes_per_update": tc["dram_read"],
    "tc_gemm_dram_write_bytes_per_update": tc["dram_write"],
    "tc_gemm_dram_bytes_per_update": tc["dram_read"] + tc["dram_write"],
    "tc_gemm_dram_bytes_per_launch": (tc["dram_read"] + tc["dram_write"]) / max(tc["launches"], 1),
    "tc_gemm_serialized_ms_per_update": tc["us"] / 1e3,
    "by_kernel": {k: dict(v, us=round(v["us"], 2)) for k, v in
                  sorted(agg.items(), key=lambda x: -x[1]["us"])},
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "by_kernel"}, indent=1))
