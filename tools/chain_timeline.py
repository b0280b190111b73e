"""Per-phase timeline of the decode layer chain inside the captured 7B decode step
(slx_decode_chain trace stamps, globaltimer ns per CTA): for every phase of a mid-step layer
chain, the spread over CTAs of (producer's first activation box issued, epilogue start =
accumulator ready / barrier passed, arrival), relative to the chain's first CTA entry; plus
the attention launches between chains.  python tools/chain_timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

cfg = LLAMA2_7B
torch.cuda.set_device(0)
lora = LoraConfig(bench.RANK, bench.ALPHA, ("q", "k", "v", "o"))
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=bench.BATCH, max_ctx=128 + 1,
                   n_slots=bench.N_ADAPTERS, max_rank=bench.RANK, max_tokens=bench.BATCH)
m.random_backbone(seed=0)
if "--bare" not in sys.argv:
    for a in range(bench.N_ADAPTERS):
        m.pool.load_random(a, lora, seed=1000 + a)
seqs = [m.alloc_seq() for _ in range(bench.BATCH)]
slots = bench.my_slots(0, 1).tolist()
sms = m._sms
n_launch = cfg.layers + 1
buf = torch.zeros(n_launch * sms * 64, dtype=torch.int64, device="cuda")
m.chain_trace = buf
dg = DecodeGraph(m, seqs, slots, fixed_pos=128).capture()
for _ in range(5):
    dg.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    dg.replay()
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1) / 20:.3f} ms (traced)")
buf.zero_()
dg.replay()
torch.cuda.synchronize()
t = buf.view(n_launch, sms, 64).cpu().numpy().astype(np.float64)
names = ["o", "post_a", "post_b", "gate_up", "down", "in_a", "in_b", "qkv", "reduce"]
prev_exit = None
acc = {}
for li in range(1, n_launch - 1):
    L = t[li]
    live = L[:, 62] > 0
    L = L[live]
    t0 = L[:, 62].min()
    ex = L[:, 63].max()
    if prev_exit is not None:
        acc.setdefault("attention (prev chain exit -> this entry)", []).append((t0 - prev_exit) / 1e3)
    acc.setdefault("chain entry spread", []).append((L[:, 62].max() - t0) / 1e3)
    for p, nm in enumerate(names):
        st, ar, px = L[:, 2 * p], L[:, 2 * p + 1], L[:, 32 + p]
        for key, col in (("x issued", px), ("start", st), ("arrive", ar)):
            v = col[col > 0]
            if len(v):
                acc.setdefault(f"{p} {nm:10s} {key:9s} min", []).append((v.min() - t0) / 1e3)
                acc.setdefault(f"{p} {nm:10s} {key:9s} max", []).append((v.max() - t0) / 1e3)
    acc.setdefault("chain exit", []).append((ex - t0) / 1e3)
    for k in (48, 49, 50, 51):   # norm item sub-stamps (debug builds)
        v = L[:, k][L[:, k] > 0]
        if len(v):
            acc.setdefault(f"norm stamp {k} med", []).append((np.median(v) - t0) / 1e3)
    prev_exit = ex
for k, v in acc.items():
    print(f"{k:48s} {np.mean(v):8.2f} us")
