"""Experiment (not product): decode GEMM (M = 64) under different stream-K grids: the default
uniform split vs all-SM stream-K (sk_ctas) for the 7B shapes; four weight copies rotate (HBM)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if os.environ.get("SLX_LIB"):   # experiment builds (exp/build_variant.sh)
    _lib.LIB_PATH = os.path.abspath(os.environ["SLX_LIB"])
from paper_2505_14468_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
shapes = {"qkv+lora": (12288 + 1536, 4096, 0), "gu": (22016, 4096, 1), "lm_head": (32000, 4096, 0)}
M = 64
for k, (n, kk, silu) in shapes.items():
    ws = [ops.pack_weight(torch.randn(n, kk, device="cuda", dtype=torch.bfloat16) * 0.02) for _ in range(4)]
    x = torch.randn(M, kk, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, n // 2 if silu else n, device="cuda", dtype=torch.bfloat16)
    ep = ops.EPI_SILU_MUL if silu else ops.EPI_NONE
    for tu in (None,):
        for i in range(3):
            ops.gemm(x, ws[i % 4], out, epilogue=ep, tuning=tu)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(40):
            ops.gemm(x, ws[i % 4], out, epilogue=ep, tuning=tu)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 40
        print(f"{os.path.basename(_lib.LIB_PATH)} {k:9s} {str(tu):10s} {us:6.1f} us  {n * kk * 2 / us / 1e3:6.0f} GB/s")
