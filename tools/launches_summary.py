"""Summarise an ncu launch list (gpu__time_duration.sum CSV): the last decode step's kernels.
python tools/launches_summary.py gpurun_out/launches.csv [kernels_per_step]"""
import collections
import csv
import sys

path = sys.argv[1]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else None
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
ids = [int(r["ID"]) for r in rows]
if per_step is None:   # one step = from the last embedding launch to the end
    starts = [i for i, r in enumerate(rows) if "embedding_kernel" in r["Kernel Name"]]
    step = rows[starts[-1]:]
else:
    step = rows[-per_step:]
cat = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in step:
    v = float(r["Metric Value"])
    us = {"ns": v / 1000, "us": v, "usecond": v, "msecond": v * 1000, "nsecond": v / 1000}.get(r["Metric Unit"], v)
    tot += us
    name = r["Kernel Name"].split("(")[0][:70] + " " + r["Grid Size"]
    cat[name][0] += 1
    cat[name][1] += us
print(f"launches in step: {len(step)}   serialized device time: {tot:.1f} us")
for k, (n, us) in sorted(cat.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:9.1f} us {n:4d}x {us / n:7.2f} us  {k}")
