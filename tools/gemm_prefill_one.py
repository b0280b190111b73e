"""One prefill-shape GEMM (13B qkv: M=16384, N=15360, K=5120, tiled W) a few times (for ncu),
and its event-timed TFLOP/s.  python tools/gemm_prefill_one.py [M N K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (16384, 15360, 5120)
a = torch.randn(M, K, device="cuda").bfloat16()
w = ops.pack_weight((torch.randn(N, K, device="cuda") * 0.02).bfloat16())
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.gemm(a, w, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ops.gemm(a, w, c)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"M={M} N={N} K={K}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")
