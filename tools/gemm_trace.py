"""Phase timeline of the decode GEMM (slx_debug_gemm_trace) for the 7B decode shapes.
python tools/gemm_trace.py [M]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib, ops  # noqa: E402
from paper_2505_14468_b200._lib import EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
DEV = "cuda"
PH = ["entry", "prolog", "pdl", "stage0", "lastmma", "accum", "red0", "exit", "red1", "seg0", "seg1", "wpass", "ld0done", "tile0done"]
lib = _lib.load()
buf = torch.zeros(4096 * 16, dtype=torch.int64, device=DEV)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
ONLY = os.environ.get("TRACE_ONLY")
for name, N, K, epi in [("qkv", 13824, 4096, EPI_NONE), ("o", 4608, 4096, EPI_RESIDUAL),
                        ("gate_up", 22016, 4096, EPI_SILU_MUL), ("down", 4096, 11008, EPI_RESIDUAL),
                        ("lm_head", 32000, 4096, EPI_NONE)]:
    if ONLY and name not in ONLY.split(","):
        continue
    a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    w = ops.pack_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
    c = torch.empty(M, N // 2 if epi == EPI_SILU_MUL else N, device=DEV, dtype=torch.bfloat16)
    r = torch.randn(M, N, device=DEV).to(torch.bfloat16) if epi == EPI_RESIDUAL else None
    for _ in range(3):
        ops.gemm(a, w, c, epilogue=epi, residual=r)
    flush.zero_()
    buf.zero_()
    torch.cuda.synchronize()
    lib.slx_debug_gemm_trace(ctypes_ptr := buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.gemm(a, w, c, epilogue=epi, residual=r)
    e1.record()
    torch.cuda.synchronize()
    lib.slx_debug_gemm_trace(None)
    t = buf.view(-1, 16).cpu().numpy().astype(np.int64)[:, :len(PH)]
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    rel[t == 0] = np.nan
    print(f"{name}: N={N} K={K} ctas={len(t)} event={e0.elapsed_time(e1) * 1000:.1f}us "
          f"span={(np.nanmax(rel)):.1f}us  GB/s(span)={N * K * 2 / np.nanmax(rel) / 1e3:.0f}")
    for i, ph in enumerate(PH):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"   {ph:8s} min {np.nanmin(col):6.2f}  p50 {np.nanmedian(col):6.2f}  max {np.nanmax(col):6.2f}")
