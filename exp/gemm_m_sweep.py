"""Experiment (not product): prefill GEMM time vs M at the 7B shapes (small merged prefills of a
serving round), against max(flops / sustained bf16 peak, weight bytes / HBM peak).  Four copies
of every weight rotate so each launch streams from HBM.  python exp/gemm_m_sweep.py [M ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
PEAK_TF, PEAK_GBS = 1389.3, 6546.6
shapes = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 0), "gu": (22016, 4096, 1), "down": (4096, 11008, 0)}
Ms = [int(a) for a in sys.argv[1:]] or [64, 128, 192, 256, 320, 400, 512, 768, 1024, 2048]
ws = {k: [ops.pack_weight(torch.randn(n, kk, device="cuda", dtype=torch.bfloat16) * 0.02) for _ in range(4)]
      for k, (n, kk, _) in shapes.items()}
tot = {}
for M in Ms:
    line = []
    for k, (n, kk, silu) in shapes.items():
        x = torch.randn(M, kk, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, n // 2 if silu else n, device="cuda", dtype=torch.bfloat16)
        ep = ops.EPI_SILU_MUL if silu else ops.EPI_NONE
        for i in range(3):
            ops.gemm(x, ws[k][i % 4], out, epilogue=ep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for i in range(reps):
            ops.gemm(x, ws[k][i % 4], out, epilogue=ep)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        ideal = max(2.0 * M * n * kk / (PEAK_TF * 1e12), n * kk * 2 / (PEAK_GBS * 1e9)) * 1e6
        line.append(f"{k} {us:7.1f} us ({ideal / us:.2f})")
        tot.setdefault(M, [0.0, 0.0])
        tot[M][0] += us
        tot[M][1] += ideal
    print(f"M={M:5d}: " + " | ".join(line) + f" | layer {tot[M][0]:.0f} us vs ideal {tot[M][1]:.0f}")
