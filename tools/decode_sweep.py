"""Decode-step variants on the config-2 workload (7B shape, 32 x r16, batch 64, ctx 128): the
same model re-captured under different host-side schedule parameters (L2 prefetch window,
split-K pieces of o / down), CUDA-graph step time per variant.
python tools/decode_sweep.py [steps] [--combos]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 30
CTX = 128
cfg = LLAMA2_7B
torch.cuda.set_device(0)
lora = LoraConfig(bench.RANK, bench.ALPHA, ("q", "k", "v", "o"))
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=bench.BATCH, max_ctx=CTX + 1,
                   n_slots=bench.N_ADAPTERS, max_rank=bench.RANK, max_tokens=bench.BATCH)
m.random_backbone(seed=0)
for a in range(bench.N_ADAPTERS):
    m.pool.load_random(a, lora, seed=1000 + a)
seqs = [m.alloc_seq() for _ in range(bench.BATCH)]
slots = bench.my_slots(0, 1).tolist()


def timed(**kw):
    saved = {k: getattr(m, k) for k in kw}
    for k, v in kw.items():
        setattr(m, k, v)
    m._pf_cache.clear()
    try:
        dg = DecodeGraph(m, seqs, slots, fixed_pos=CTX).capture()
        for _ in range(5):
            dg.replay()
        torch.cuda.synchronize()
        best = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                dg.replay()
            e1.record()
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1) / steps)
        del dg
        return min(best)
    finally:
        for k, v in saved.items():
            setattr(m, k, v)
        m._pf_cache.clear()


variants = [{}]
if "--combos" in sys.argv:
    for mb in (8.0, 12.0, 16.0):
        variants.append({"l2_prefetch_mb": mb})
    variants.append({})
else:
    for mb in (0.0, 8.0, 24.0, 32.0, 48.0):
        variants.append({"l2_prefetch_mb": mb})
    for so in (4, 5, 7, 8):
        variants.append({"splitk_splits_o": so})
    for sd in (6, 7, 9):
        variants.append({"splitk_splits_dn": sd})
for v in variants:
    ms = timed(**v)
    print(json.dumps({"variant": v, "ms_per_step": round(ms, 4),
                      "tokens_per_s": round(bench.BATCH / ms * 1000.0, 1)}), flush=True)
