"""DRAM traffic per launch of the decode-step kernels from an ncu CSV with
dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum (one bench step = the last
`per_step` launches).  Writes profiles/traffic.json for bench.py's roofline.traffic.
python tools/ncu_traffic.py gpurun_out/traffic.csv [per_step]"""
import collections
import csv
import json
import os
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
by_id = collections.OrderedDict()
for r in rows:
    d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"]})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
             "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
    d[r["Metric Name"]] = v * scale
launches = list(by_id.values())
gemm = [x for x in launches if "gemm_sk_kernel" in x["name"]]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 129
step = gemm[-per_step:]
tot = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in step)
out = {"gemm_sk_kernel_bytes_per_launch": tot / len(step), "launches": len(step),
       "gemm_sk_kernel_us_per_launch_serialised": sum(x["gpu__time_duration.sum"] for x in step) / len(step),
       "by_grid": {}}
for x in step:
    g = out["by_grid"].setdefault(x["grid"], {"n": 0, "dram_bytes": 0.0, "us": 0.0})
    g["n"] += 1
    g["dram_bytes"] += x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"]
    g["us"] += x["gpu__time_duration.sum"]
for g in out["by_grid"].values():
    g["dram_bytes"] /= g["n"]
    g["us"] /= g["n"]
attn = [x for x in launches if "attn" in x["name"]][-32:]
if attn:
    out["attn_decode_bytes_per_launch"] = sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in attn) / len(attn)
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(os.path.join("profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
