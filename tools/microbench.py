"""Per-kernel timing of the decode-step kernels at config-2 shapes (CUDA events, L2 flushed
between iterations).  Usage: python tools/microbench.py [gemm|lora|attn|all]"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200._lib import EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL  # noqa: E402

DEV = "cuda"
PEAK = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6537.3) if os.path.exists("MEASURED_PEAKS.json") else 6537.3
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)


def timeit(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush_buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def gemm_shapes(M=64):
    out = []
    for name, N, K, epi in [("qkv", 12288, 4096, EPI_NONE), ("o", 4096, 4096, EPI_RESIDUAL),
                            ("gate_up", 22016, 4096, EPI_SILU_MUL), ("down", 4096, 11008, EPI_RESIDUAL),
                            ("lm_head", 32000, 4096, EPI_NONE)]:
        a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
        w = ops.pack_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
        nout = N // 2 if epi == EPI_SILU_MUL else N
        c = torch.empty(M, nout, device=DEV, dtype=torch.bfloat16)
        r = torch.randn(M, N, device=DEV).to(torch.bfloat16) if epi == EPI_RESIDUAL else None
        ms = timeit(lambda: ops.gemm(a, w, c, epilogue=epi, residual=r))
        byts = N * K * 2 + M * K * 2 + M * nout * 2 * (2 if r is not None else 1)
        gbs = byts / ms / 1e6
        out.append({"gemm": name, "M": M, "N": N, "K": K, "us": round(ms * 1000, 2),
                    "GB/s": round(gbs, 1), "frac": round(gbs / PEAK, 3)})
    return out


def lora_shapes():
    from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig
    from paper_2505_14468_b200.model import AdapterPool
    import numpy as np
    cfg = LLAMA2_7B
    pool = AdapterPool(cfg, ("q", "k", "v", "o"), 32, 16, DEV)
    from dataclasses import replace
    one = replace(cfg, layers=1)
    pool = AdapterPool(one, ("q", "k", "v", "o"), 32, 16, DEV)
    for a in range(32):
        pool.load_random(a, LoraConfig(16, 32.0, ("q", "k", "v", "o")), seed=a)
    B = 64
    slots = torch.from_numpy(np.random.default_rng(0).integers(0, 32, size=B).astype(np.int32)).to(DEV)
    distinct = len(set(slots.tolist()))
    x = torch.randn(B, 4096, device=DEV).to(torch.bfloat16)
    y = torch.randn(B, 12288, device=DEV).to(torch.bfloat16)
    ws = torch.zeros(ops.lora_workspace_bytes(B, 32, 16, 3), dtype=torch.uint8, device=DEV)
    ops.lora_plan_tokens(slots, 32, ws)
    tg = ops.make_targets([(pool.a_ptr[0, i], pool.b_ptr[0, i], 4096, 4096 * i, 4096, 4096) for i in range(3)])
    ms = timeit(lambda: ops.lora_apply(y, x, 4096, pool.rank, pool.scale, 16, tg, ws))
    byts = 3 * (distinct * 16 * (4096 + 4096) * 2 + B * 4096 * 2 + 2 * B * 4096 * 2)
    return [{"lora": "qkv", "distinct": distinct, "us": round(ms * 1000, 2), "GB/s": round(byts / ms / 1e6, 1),
             "frac": round(byts / ms / 1e6 / PEAK, 3)}]


def attn_shapes():
    B, H, D, ctx = 64, 32, 128, 128
    kc = torch.randn(B, H, ctx + 1, D, device=DEV).to(torch.bfloat16)
    vc = torch.randn_like(kc)
    qkv = torch.randn(B, 3 * H * D, device=DEV).to(torch.bfloat16)
    out = torch.empty(B, H * D, device=DEV, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=DEV)
    seq = torch.arange(B, dtype=torch.int32, device=DEV)
    ms = timeit(lambda: ops.attention(out, qkv, H, H, D, pos, seq, kc, vc))
    byts = B * (ctx + 1) * 2 * H * D * 2
    return [{"attn": "decode", "us": round(ms * 1000, 2), "GB/s": round(byts / ms / 1e6, 1),
             "frac": round(byts / ms / 1e6 / PEAK, 3)}]


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    res = []
    if what in ("gemm", "all"):
        res += gemm_shapes()
    if what in ("lora", "all"):
        res += lora_shapes()
    if what in ("attn", "all"):
        res += attn_shapes()
    for r in res:
        print(json.dumps(r))
