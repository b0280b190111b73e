"""Stall samples of an ncu report attributed to source-line ranges of one file, walking the SASS
in address order (inlined helpers count toward the enclosing line of `file`).
python tools/phase_hot.py report.ncu-rep file.cu name:lo-hi [name:lo-hi ...]"""
import csv
import io
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
phases = []
for spec in sys.argv[3:]:
    n, r = spec.split(":")
    lo, hi = map(int, r.split("-"))
    phases.append((n, lo, hi))


def ncu(mode):
    return subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode,
                           "--launch-count", "1"], capture_output=True, text=True).stdout


addr_line, cur, f = {}, None, None
for row in csv.reader(io.StringIO(ncu("cuda,sass"))):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:
        cur = (f, int(row[0]))
        continue
    if len(row) > 2 and row[2].startswith("0x"):
        addr_line[int(row[2], 16)] = cur
rows = list(csv.reader(io.StringIO(ncu("sass"))))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
seen, last, agg, tot = set(), None, {}, 0.0
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr) or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    if a in seen:
        continue
    seen.add(a)
    fl = addr_line.get(a)
    if fl and fl[0] == fname:
        last = fl[1]
    v = float(r[i_s] or 0)
    tot += v
    ph = next((n for n, lo, hi in phases if last is not None and lo <= last <= hi), "other")
    agg[ph] = agg.get(ph, 0.0) + v
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:12s} {v:7.0f} {100 * v / max(tot, 1):5.1f}%")
