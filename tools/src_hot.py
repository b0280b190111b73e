"""Stall samples per CUDA source line of an ncu report (needs -lineinfo + --import-source).
python tools/src_hot.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
agg, fname, total = {}, None, 0.0
cur = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:   # a source line row: remember it; sass rows follow with empty first column
        cur = (fname, int(row[0]), row[1].strip()[:90])
        continue
    if len(row) > 4 and cur:
        try:
            v = float(row[4])
        except ValueError:
            continue
        agg[cur] = agg.get(cur, 0.0) + v
        total += v
print("samples", total)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:7.0f} {100 * v / max(total, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
