"""Run the config-2 decode attention a few times (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402

DEV = "cuda"
B, H, D, ctx = 64, 32, 128, 128
kc = torch.randn(B, H, ctx + 1, D, device=DEV).to(torch.bfloat16)
vc = torch.randn_like(kc)
qkv = torch.randn(B, 3 * H * D, device=DEV).to(torch.bfloat16)
out = torch.empty(B, H * D, device=DEV, dtype=torch.bfloat16)
pos = torch.full((B,), ctx, dtype=torch.int32, device=DEV)
seq = torch.arange(B, dtype=torch.int32, device=DEV)
for _ in range(5):
    ops.attention(out, qkv, H, H, D, pos, seq, kc, vc)
torch.cuda.synchronize()
