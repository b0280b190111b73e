"""Summarise an ncu launch list of one config-3 prefill forward (gpu__time_duration,
sm__pipe_tensor_cycles_active %, dram__bytes_read/write per launch; tools/ncu_prefill.sh):
per kernel and grid, launches, mean duration, tensor-pipe share and DRAM bytes per launch, plus
the GEMM totals against their algorithmic bytes.  Writes profiles/prefill_traffic.json (read by
bench.py's config-3 roofline.traffic).
python tools/prefill_launches_summary.py gpurun_out/prefill_launches.csv"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
by_id = collections.OrderedDict()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
         "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "%": 1}
for r in rows:
    d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
agg = collections.OrderedDict()
for d in by_id.values():
    k = (d["name"][:60], d["grid"])
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    a[3] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
print(f"{'launches':>8s} {'us/launch':>10s} {'tensor%':>8s} {'DRAM MB/launch':>15s}  kernel grid")
for (name, grid), (n, us, tp, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {us / n:10.1f} {tp / n:8.1f} {by / n / 1e6:15.1f}  {name} {grid}")
gemm = [d for d in by_id.values() if "gemm_tc" in d["name"]]
tot_us = sum(d.get("gpu__time_duration.sum", 0.0) for d in gemm)
tot_b = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in gemm)
tp = (sum(d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0) *
          d.get("gpu__time_duration.sum", 0.0) for d in gemm) / tot_us) if tot_us else 0.0
out = {"gemm_tc_launches": len(gemm), "gemm_tc_us_serialised": tot_us,
       "gemm_tc_tensor_pipe_pct_time_weighted": tp, "gemm_tc_dram_bytes_per_launch": tot_b / max(1, len(gemm))}
print(json.dumps(out))
json.dump(out, open(os.path.join(ROOT, "profiles", "prefill_traffic.json"), "w"), indent=1)
