"""Run the config-2 q/k/v LoRA apply a few times (for ncu)."""
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import AdapterPool  # noqa: E402

DEV = "cuda"
one = replace(LLAMA2_7B, layers=1)
pool = AdapterPool(one, ("q", "k", "v", "o"), 32, 16, DEV)
for a in range(32):
    pool.load_random(a, LoraConfig(16, 32.0, ("q", "k", "v", "o")), seed=a)
B = 64
slots = torch.from_numpy(np.random.default_rng(0).integers(0, 32, size=B).astype(np.int32)).to(DEV)
x = torch.randn(B, 4096, device=DEV).to(torch.bfloat16)
y = torch.randn(B, 12288, device=DEV).to(torch.bfloat16)
ws = torch.zeros(ops.lora_workspace_bytes(B, 32, 16, 3), dtype=torch.uint8, device=DEV)
ops.lora_plan_tokens(slots, 32, ws)
tg = ops.make_targets([(pool.a_ptr[0, i], pool.b_ptr[0, i], 4096, 4096 * i, 4096, 4096) for i in range(3)])
for _ in range(5):
    ops.lora_apply(y, x, 4096, pool.rank, pool.scale, 16, tg, ws)
torch.cuda.synchronize()
