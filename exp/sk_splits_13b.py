"""Experiment (not product): 13B decode step vs the split-K piece counts of the o / down
projections (o: 20 tiles x S_o CTAs, down: 20 x S_dn; one tcgen05 CTA per SM, 148 SMs), on the
config-3 adapter pool (gathered LoRA) and the bare backbone.  python exp/sk_splits_13b.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

B, CTX, NS = 64, 128, 128
cfg = LLAMA2_13B
torch.cuda.set_device(0)
ranks = np.random.default_rng(0).choice([8, 16, 64], size=NS)
slots = np.random.default_rng(0).integers(0, NS, size=B).astype(np.int32)
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=B, max_ctx=CTX + 1, n_slots=NS,
                   max_rank=64, max_tokens=B, lora_targets=("q", "k", "v", "o"))
m.random_backbone(seed=0)
for a in range(NS):
    m.pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
seqs = [m.alloc_seq() for _ in range(B)]


def step_ms(slot_list, n=20):
    dg = DecodeGraph(m, seqs, slot_list, fixed_pos=CTX)
    dg.capture()
    for _ in range(5):
        dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        dg.replay()
    e1.record()
    torch.cuda.synchronize()
    del dg
    return e0.elapsed_time(e1) / n


for so, sdn in [(6, 8), (4, 5)]:
    m.splitk_splits_o, m.splitk_splits_dn = so, sdn
    lo = step_ms(slots.tolist())
    bare = step_ms([-1] * B)
    print(f"S_o {so} S_dn {sdn}: pool step {lo:.3f} ms, no-adapter tokens {bare:.3f} ms", flush=True)
