"""Experiment (not product): CUDA-graph decode step vs batch size on the config-2 model (7B shape,
32 x r16 adapters on q,k,v,o, ctx 128).  python exp/decode_batch.py [B ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if os.environ.get("SLX_LIB"):   # experiment builds (exp/build_variant.sh)
    _lib.LIB_PATH = os.path.abspath(os.environ["SLX_LIB"])
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

Bs = [int(a) for a in sys.argv[1:]] or [64, 96, 128]
CTX, NA = 128, 32
torch.cuda.set_device(0)
lora = LoraConfig(16, 32.0, ("q", "k", "v", "o"))
m = MultiLoraModel(LLAMA2_7B, dtype=torch.bfloat16, max_seqs=max(Bs), max_ctx=CTX + 1, n_slots=NA,
                   max_rank=16, max_tokens=max(Bs))
m.random_backbone(seed=0)
for a in range(NA):
    m.pool.load_random(a, lora, seed=1000 + a)
rng = np.random.default_rng(0)
for B in Bs:
    seqs = [m.alloc_seq() for _ in range(B)]
    dg = DecodeGraph(m, seqs, rng.integers(0, NA, size=B).tolist(), fixed_pos=CTX).capture()
    for _ in range(5):
        dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        dg.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    print(f"batch {B}: {ms:.3f} ms/step, {B / ms * 1e3:.0f} tokens/s, fast path {m._decode_fast(B)}")
    del dg
    for s_ in seqs:
        m.free_seq(s_)

# per-kernel-family device time of one eager decode step at each batch (ops.KernelTimer)
from paper_2505_14468_b200 import ops  # noqa: E402

for B in Bs:
    seqs = [m.alloc_seq() for _ in range(B)]
    for s_ in seqs:
        m.seq_len[s_] = CTX
    slots = rng.integers(0, NA, size=B).tolist()
    toks = rng.integers(1, 32000, size=B).tolist()
    m.decode(seqs, toks, slots)
    for s_ in seqs:
        m.seq_len[s_] = CTX
    torch.cuda.synchronize()
    with ops.KernelTimer() as kt:
        torch.cuda._sleep(50_000_000)
        m.decode(seqs, toks, slots)
    torch.cuda.synchronize()
    print(B, {k: (round(v[0], 3), v[1]) for k, v in kt.durations().items()})
    for s_ in seqs:
        m.free_seq(s_)
