"""Decode-step time (CUDA graph replay, device events) of the bench workload under variants, to
attribute in-graph time: python tools/step_variants.py [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200._lib import load  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
load()
cfg = LLAMA2_7B
lora = LoraConfig(bench.RANK, bench.ALPHA, ("q", "k", "v", "o"))
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=bench.BATCH, max_ctx=bench.CTX + 1,
                   n_slots=bench.N_ADAPTERS, max_rank=bench.RANK, max_tokens=bench.BATCH)
m.random_backbone(seed=0)
for a in range(bench.N_ADAPTERS):
    m.pool.load_random(a, lora, seed=1000 + a)
g = torch.Generator(device=m.device).manual_seed(7)
for l in range(cfg.layers):
    m.k_cache[l].normal_(generator=g)
    m.v_cache[l].normal_(generator=g)
seqs = [m.alloc_seq() for _ in range(bench.BATCH)]
slots = bench.tok_slots()


def timed(slot_list, stacked=True, fuse=True):
    m.use_stacked_decode, m.fuse_expand = stacked, fuse
    dg = DecodeGraph(m, seqs, slot_list, fixed_pos=bench.CTX)
    dg.tok.copy_(torch.randint(1, cfg.vocab, (bench.BATCH,), generator=g, device=m.device,
                               dtype=torch.int32))
    dg.capture()
    for _ in range(3):
        dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dg.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return ms, dg.kernels_per_step


none = [-1] * bench.BATCH
# prefetch configurations, interleaved over rounds (box-to-box variance is larger than the effects)
cfgs = []
for spec in [x for x in os.environ.get("PF_SWEEP", "").split(";") if x]:
    mb, early, last, wo_all = spec.split(",")
    cfgs.append((float(mb), early, last, wo_all == "1"))
if cfgs:
    graphs = []
    for mb, early, last, wo_all in cfgs:
        os.environ["SLX_ATTN_PF_EARLY"], os.environ["SLX_PF_EVICT_LAST"] = early, last
        m.l2_prefetch_mb, m._pf_cache = mb, {}
        if not wo_all:
            m._pf_all = lambda key, t: m._pf(key, t)
        else:
            m.__dict__.pop("_pf_all", None)
        m.use_stacked_decode, m.fuse_expand = True, True
        dg = DecodeGraph(m, seqs, slots.tolist(), fixed_pos=bench.CTX)
        dg.capture()
        graphs.append(((mb, early, last, wo_all), dg))
    res = {c: [] for c, _ in graphs}
    for _ in range(3):
        for c, dg in graphs:
            for _ in range(3):
                dg.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                dg.replay()
            e1.record()
            torch.cuda.synchronize()
            res[c].append(e0.elapsed_time(e1) / steps)
    for c, v in res.items():
        print(f"prefetch mb={c[0]:5.1f} attn_early={c[1]} evict_last={c[2]} wo_all={c[3]}: "
              f"{min(v):7.3f} ms/step  {bench.BATCH / min(v) * 1000:9.0f} tok/s", flush=True)
    sys.exit(0)
m.l2_prefetch_mb, m._pf_cache = float(os.environ.get("SLX_L2_PF_MB", "32")), {}
for name, args in [("lora fused", (slots.tolist(), True, True)),
                   ("lora expand kernels", (slots.tolist(), True, False)),
                   ("lora shrink/expand kernels (no stacking)", (slots.tolist(), False, False)),
                   ("no adapters, stacked rows", (none, True, True)),
                   ("no adapters, no stacked rows", (none, False, False))]:
    ms, k = timed(*args)
    print(f"{name:45s} {ms:7.3f} ms/step  {bench.BATCH / ms * 1000:9.0f} tok/s  kernels {k}", flush=True)
