"""Top stall-sampled SASS instructions of an ncu report (first kernel or -k index).
python tools/sass_hot.py report.ncu-rep [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr) and r[0] != "Address"]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
val = lambda r: float(r[i_s] or 0)  # noqa: E731
tot = sum(val(r) for r in data)
print(rows[0][1][:120] if rows and len(rows[0]) > 1 else "", "samples", tot)
for r in sorted(data, key=lambda r: -val(r))[:top]:
    print(f"{val(r):7.0f} {100 * val(r) / max(tot, 1):5.1f}%  {r[0]}  {r[1][:100]}")
