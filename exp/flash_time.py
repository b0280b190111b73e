"""Experiment harness (not product): time slx_attention_prefill on the config-3 layer shape
(8 x 2048-token causal segments, 40 heads, head_dim 128) from a given libslora_b200 build.
python exp/flash_time.py [path/to/lib.so]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_2505_14468_b200 import ops  # noqa: E402

torch.cuda.set_device(0)
H, D, P, L = 40, 128, 8, 2048
dev = "cuda"
qkv = torch.randn(P * L, 3 * H * D, device=dev).to(torch.bfloat16)
kc = torch.randn(P, H, L, D, device=dev).to(torch.bfloat16)
vc = torch.randn(P, H, L, D, device=dev).to(torch.bfloat16)
out = torch.empty(P * L, H * D, device=dev, dtype=torch.bfloat16)
plan = ops.prefill_plan([(i * L, L, i, 0) for i in range(P)], H, dev)
order = os.environ.get("FLASH_ORDER", "cost")
if order != "cost":   # experiment: item order by (segment, head), costliest pair first
    t_cpu, it_cpu = plan[0].cpu(), plan[1].cpu().tolist()
    seq = t_cpu[:, 2].tolist()
    if order == "head":
        it_cpu.sort(key=lambda it: (seq[it[0]], it[2], -it[0]))
    elif order == "head_interleave":   # heads of a segment interleaved with costs descending
        it_cpu.sort(key=lambda it: (seq[it[0]], -it[0], it[2]))
    plan = (plan[0], torch.tensor(it_cpu, dtype=torch.int32, device=dev))
for _ in range(3):
    ops.attention_prefill(out, qkv, H, H, D, plan, kc, vc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ops.attention_prefill(out, qkv, H, H, D, plan, kc, vc)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 100.0
flops = P * (L * (L + 1) // 2) * 4 * D * H
print(f"{os.path.basename(_lib.LIB_PATH)} order={order}: {us:.1f} us/layer  {flops / us / 1e6:.1f} TFLOP/s")
if "dbg" in _lib.LIB_PATH:
    import ctypes
    import numpy as np
    lib = _lib.load()
    buf = np.zeros(8192, dtype=np.uint64)
    lib.slx_dbg_copy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(8192 * 8))
    st = buf.reshape(1024, 8)[:400].astype(np.int64)
    d = np.diff(st[:, 0])
    print("block period (clk) median", np.median(d[1:300]), "mean", d[1:300].mean())
    tokw = st[1:300, 5] - st[1:300, 2]
    print("  token wait     median", np.median(tokw), "mean", tokw.mean(), "(0 if no token build)")
    for name, a, b in (("wait S", 0, 1), ("tmem ld", 1, 2), ("compute", 2, 3), ("P store+fence", 3, 4), ("arrive->next", 4, 0)):
        if name == "arrive->next":
            v = st[1:300, 0] - st[0:299, 4]
        else:
            v = st[1:300, b] - st[1:300, a]
        print(f"  {name:14s} median {np.median(v):8.0f} mean {v.mean():8.0f}")
