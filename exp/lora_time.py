"""Experiment harness (not product): time the gathered decode shrink and expand at the config-3
pool (13B widths, 128 slots r{8,16,64}, batch 64, q/k/v targets) from a given build."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import AdapterPool  # noqa: E402

torch.cuda.set_device(0)
cfg, B, NS = LLAMA2_13B, 64, 128
dev = torch.device("cuda")
pool = AdapterPool(cfg, ("q", "k", "v", "o"), NS, 64, dev)
ranks = np.random.default_rng(0).choice([8, 16, 64], size=NS)
for a in range(NS):
    pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
slots = torch.from_numpy(np.random.default_rng(0).integers(0, NS, size=B).astype(np.int32)).to(dev)
ws = torch.zeros(ops.lora_workspace_bytes(B, NS, 64, 4) + 256, dtype=torch.uint8, device=dev)
ops.lora_plan_tokens(slots, NS, ws)
d = cfg.hidden
x = torch.randn(B, d, device=dev).to(torch.bfloat16)
qkv = torch.randn(B, 3 * d, device=dev).to(torch.bfloat16)
v = torch.zeros(B, 3 * 64, device=dev)
specs = [(pool.a_ptr[0, i], pool.b_ptr[0, i], d, i * d, d, d) for i in range(3)]
tg = ops.make_targets(specs)
offs = [0, 64, 128]


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


us_s = t(lambda: ops.lora_shrink(v, x, pool.rank, 64, tg, offs, ws))
us_e = t(lambda: ops.lora_expand(qkv, v, pool.rank, pool.scale, 64, tg, offs, ws, v_slot_stride=0))
print(f"{os.path.basename(_lib.LIB_PATH)}: shrink {us_s:.1f} us, expand {us_e:.1f} us (q/k/v, 13B, 128-slot pool)")
