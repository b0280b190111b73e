"""Run the 7B-shape decode attention (pipelined, fused LoRA delta) a few times (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.model import rope_tables  # noqa: E402
from paper_2505_14468_b200 import ops  # noqa: E402

DEV = "cuda"
B, H, D, CTX, R, NS = 64, 32, 128, 128, 16, 32
cos, sin = rope_tables(CTX + 8, D, 10000.0)
cos_d, sin_d = torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV)
kc = torch.randn(B, H, CTX + 1, D, device=DEV).bfloat16()
vc = torch.randn(B, H, CTX + 1, D, device=DEV).bfloat16()
qkv = torch.randn(B, 3 * H * D, device=DEV).bfloat16()
out = torch.empty(B, H * D, device=DEV, dtype=torch.bfloat16)
pos = torch.full((B,), CTX, dtype=torch.int32, device=DEV)
seq = torch.arange(B, dtype=torch.int32, device=DEV)
slot = torch.from_numpy(np.random.default_rng(0).integers(0, NS, size=B).astype(np.int32)).to(DEV)
ranks = torch.full((NS,), R, dtype=torch.int32, device=DEV)
scales = torch.full((NS,), 2.0, device=DEV)
v_all = torch.randn(B, 3 * NS * R, device=DEV)
Bs = [torch.randn(NS, H * D, R, device=DEV).bfloat16() for _ in range(3)]
tabs = [torch.tensor([b[s].data_ptr() for s in range(NS)], dtype=torch.int64, device=DEV) for b in Bs]
delta = ops.make_delta(v_all, slot, ranks, scales, R, [(tabs[i], i * NS * R, i * H * D, H * D) for i in range(3)])
lora = os.environ.get("LORA", "1") == "1"
for _ in range(5):
    ops.rope_attention_decode(out, qkv, H, H, D, pos, seq, cos_d, sin_d, kc, vc, lora=delta if lora else None)
torch.cuda.synchronize()
