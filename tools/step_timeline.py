"""In-graph timeline of the decode step: GEMM and attention launches record globaltimer stamps
(slx_debug_gemm_trace windows); prints per launch the first CTA entry, first data, last CTA exit
relative to the step start and the gap to the next traced launch.  python tools/step_timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200 import _lib  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

lib = _lib.load()
cfg = LLAMA2_7B
lora = LoraConfig(bench.RANK, bench.ALPHA, ("q", "k", "v", "o"))
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=bench.BATCH, max_ctx=128 + 1,
                   n_slots=bench.N_ADAPTERS, max_rank=bench.RANK, max_tokens=bench.BATCH)
m.random_backbone(seed=0)
for a in range(bench.N_ADAPTERS):
    m.pool.load_random(a, lora, seed=1000 + a)
seqs = [m.alloc_seq() for _ in range(bench.BATCH)]
dg = DecodeGraph(m, seqs, bench.my_slots(0, 1).tolist(), fixed_pos=128)
dg.capture()      # untraced warm-up / plans
buf = torch.zeros(200 * 4096, dtype=torch.int64, device="cuda")
lib.slx_debug_gemm_trace(buf.data_ptr())
dgt = DecodeGraph(m, seqs, bench.my_slots(0, 1).tolist(), fixed_pos=128)
dgt.capture()
lib.slx_debug_gemm_trace(None)
for _ in range(3):
    dgt.replay()
torch.cuda.synchronize()
dgt.replay()
torch.cuda.synchronize()
t = buf.view(200, 4096).cpu().numpy()
names = {1: "gemm", 2: "gemm+res", 3: "gemm+silu", 4: "gemm-splitk", 5: "attention", 6: "rmsnorm"}
rows = []
stamps = []
for i in range(200):
    kind = int(t[i, 4095] & 0xffffffff)
    if kind == 0:
        continue
    st = t[i, :4095 - 15].reshape(-1, 16)
    st = st[st[:, 0] > 0]
    if len(st) == 0:
        continue
    entry = st[:, 0].min()
    if kind == 5:
        exit_ = max(st[:, 7].max(), st[:, 8].max())
        first = st[:, 2][st[:, 2] > 0].min() if (st[:, 2] > 0).any() else entry
    elif kind == 6:
        exit_ = st[:, 7].max()
        first = st[:, 2].max()   # last CTA past the PDL wait
    else:   # GEMMs: thread 0 stamps 7 before the epilogue warps finish (stamp 8)
        exit_ = max(st[:, 7].max(), st[:, 8].max())
        first = st[:, 3][st[:, 3] > 0].min() if (st[:, 3] > 0).any() else entry
    rows.append((names.get(kind, str(kind)), entry, first, exit_, len(st)))
    stamps.append(st)
rows = rows[-(7 * cfg.layers + 2):]
stamps = stamps[-len(rows):]   # the captured graph's launches (warm-up windows come first)
t0 = rows[0][1]
prev_end = None
tot = {}
print(f"{'kernel':12s} {'ctas':>5s} {'start':>9s} {'1st data':>9s} {'end':>9s} {'dur':>7s} {'gap':>7s}")
for name, e, f, x, n in rows[:22]:
    gap = (e - prev_end) / 1000 if prev_end is not None else 0.0
    print(f"{name:12s} {n:5d} {(e - t0) / 1000:9.2f} {(f - t0) / 1000:9.2f} {(x - t0) / 1000:9.2f} "
          f"{(x - e) / 1000:7.2f} {gap:7.2f}")
    prev_end = x
gaps = {}
for i, (name, e, f, x, n) in enumerate(rows):
    d = tot.setdefault(name, [0, 0.0, 0.0])
    d[0] += 1
    d[1] += (x - e) / 1000
    d[2] += (f - e) / 1000
    if i + 1 < len(rows):
        gaps.setdefault((name, rows[i + 1][0]), []).append(((rows[i + 1][1] - x) / 1000,
                                                             (rows[i + 1][2] - x) / 1000))
print("step span (first entry -> last exit):", (rows[-1][3] - t0) / 1000, "us")
# fused-norm prologue phases (GEMM windows with stamps 10..14)
ph = {}
for i in range(200):
    kind = int(t[i, 4095] & 0xffffffff)
    if kind not in (1, 2, 3):
        continue
    st = t[i, :4095 - 15].reshape(-1, 16)
    st = st[st[:, 0] > 0]
    if len(st) == 0 or not (st[:, 10] > 0).any():
        continue
    e = st[:, 0].min()
    for k in (10, 11, 12, 13, 14, 2):
        col = st[:, k][st[:, k] > 0]
        ph.setdefault((kind, k), []).append(((col.min() - e) / 1000, (col.max() - e) / 1000))
for (kind, k), v in sorted(ph.items()):
    v = np.array(v)
    print(f"  prologue kind {kind} stamp {k:2d}: min {v[:, 0].mean():7.2f}  max {v[:, 1].mean():7.2f} us after entry")
# critical-path share: exit-to-exit time attributed to each launch, split into
# (previous exit -> this first data) and (this first data -> this exit)
cp = {}
for i in range(1, len(rows)):
    key = (rows[i - 1][0], rows[i][0])
    d = cp.setdefault(key, [0, 0.0, 0.0])
    d[0] += 1
    d[1] += (rows[i][2] - rows[i - 1][3]) / 1000
    d[2] += (rows[i][3] - rows[i][2]) / 1000
tot_cp = 0.0
for (a, b), (n, w, r) in cp.items():
    print(f"  exit-to-exit {a:>12s} -> {b:12s}: {(w + r) / n:7.2f} us = wait {w / n:6.2f} + run {r / n:6.2f}  (x{n})")
    tot_cp += w + r
print(f"  sum of exit-to-exit: {tot_cp:.1f} us")
# per dependent launch: stamps 0..8 (min / median / max over CTAs) relative to the previous exit
det = {}
for i in range(1, len(rows)):
    key = (rows[i - 1][0], rows[i][0])
    st = stamps[i]
    prev_exit = rows[i - 1][3]
    acc = det.setdefault(key, {})
    for k in range(9):
        col = st[:, k][st[:, k] > 0]
        if len(col):
            acc.setdefault(k, []).append(((col.min() - prev_exit) / 1000, np.median(col - prev_exit) / 1000,
                                          (col.max() - prev_exit) / 1000))
for (a, b), acc in det.items():
    print(f"  stamps of {b} after {a} exit (min/med/max over CTAs, us):")
    for k, v in sorted(acc.items()):
        v = np.array(v).mean(axis=0)
        print(f"     stamp {k}: {v[0]:8.2f} {v[1]:8.2f} {v[2]:8.2f}")
for k, (n, us, fd) in tot.items():
    print(f"  {k:12s} {n:3d} launches, mean entry->exit {us / n:7.2f} us, entry->first data {fd / n:6.2f} us")
for (a, b), v in gaps.items():
    v = np.array(v)
    print(f"  gap {a:>12s} -> {b:12s}: entry {v[:, 0].mean():7.2f} us, first data {v[:, 1].mean():7.2f} us "
          f"after this exit")
