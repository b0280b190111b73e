"""Decode attention (7B shape: 64 tokens x 32 heads x D 128, ctx 128) timed as a CUDA graph of
back-to-back launches over 3 KV pools (> L2), with and without the fused LoRA delta.  python tools/attn_bench.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 2:   # experiment builds: python tools/attn_bench.py reps path/to/lib.so
    _lib.LIB_PATH = os.path.abspath(sys.argv[2])
from paper_2505_14468_b200.model import rope_tables  # noqa: E402
from paper_2505_14468_b200 import ops  # noqa: E402

DEV = "cuda"
REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 30
B, H, D, CTX, R, NS = 64, 32, 128, int(os.environ.get("CTX", 128)), 16, 32
cos, sin = rope_tables(CTX + 8, D, 10000.0)
cos_d, sin_d = torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV)
pools = [(torch.randn(B, H, CTX + 1, D, device=DEV).bfloat16(),
          torch.randn(B, H, CTX + 1, D, device=DEV).bfloat16()) for _ in range(3)]
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
kv_bytes = B * H * CTX * D * 2 * 2


def run(lora):
    def body():
        for i in range(REPS):
            kc, vc = pools[i % 3]
            ops.rope_attention_decode(out, qkv, H, H, D, pos, seq, cos_d, sin_d, kc, vc,
                                      lora=delta if lora else None)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000 / REPS)
    us = sorted(ts)[2]
    return {"lora": lora, "ctx": CTX, "us": round(us, 2), "GB/s": round(kv_bytes / us / 1e3, 1)}


for lora in (False, True):
    print(json.dumps(run(lora)), flush=True)
