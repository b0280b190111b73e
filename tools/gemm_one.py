"""Run one decode GEMM shape a few times (for ncu).  python tools/gemm_one.py N K [epi] [M]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
epi = int(sys.argv[3]) if len(sys.argv) > 3 else 0
M = int(sys.argv[4]) if len(sys.argv) > 4 else 64
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = ops.pack_weight((torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16))
r = torch.randn(M, N, device="cuda").to(torch.bfloat16) if epi == 1 else None
for _ in range(5):
    ops.gemm(a, w, epilogue=epi, residual=r)
torch.cuda.synchronize()
