"""Experiment (not product): gathered shrink / expand time at prefill token counts (7B widths,
24 r16 slots, q/k/v targets, contiguous same-adapter segments).  python exp/lora_prefill_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import AdapterPool  # noqa: E402

torch.cuda.set_device(0)
cfg, NS = LLAMA2_7B, 24
dev = torch.device("cuda")
pool = AdapterPool(cfg, ("q", "k", "v", "o"), NS, 16, dev)
for a in range(NS):
    pool.load_random(a, LoraConfig(16, 32.0), seed=100 + a)
d = cfg.hidden


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


for T, nseg in ((64, 4), (256, 4), (480, 8), (512, 4), (1024, 8)):
    slots = torch.from_numpy(np.repeat(np.arange(nseg), T // nseg).astype(np.int32)).to(dev)
    ws = torch.zeros(ops.lora_workspace_bytes(T, NS, 16, 4) + 256, dtype=torch.uint8, device=dev)
    ops.lora_plan_tokens(slots, NS, ws)
    x = torch.randn(T, d, device=dev).to(torch.bfloat16)
    qkv = torch.randn(T, 3 * d, device=dev).to(torch.bfloat16)
    v = torch.zeros(T, 3 * 16, device=dev)
    specs = [(pool.a_ptr[0, i], pool.b_ptr[0, i], d, i * d, d, d) for i in range(3)]
    tg = ops.make_targets(specs)
    offs = [0, 16, 32]
    us_s = t(lambda: ops.lora_shrink(v, x, pool.rank, 16, tg, offs, ws))
    us_e = t(lambda: ops.lora_expand(qkv, v, pool.rank, pool.scale, 16, tg, offs, ws, v_slot_stride=0))
    print(f"T={T} ({nseg} segs): shrink {us_s:.1f} us, expand {us_e:.1f} us (q/k/v)")
