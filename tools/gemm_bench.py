"""Decode GEMM shapes (7B, M tokens) timed as a CUDA graph of back-to-back launches (PDL
chained, weights rotated over 3 copies so nothing is served from L2), stream-K vs the
cluster/global split-K path.  python tools/gemm_bench.py [M] [reps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200._lib import EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL  # noqa: E402

DEV = "cuda"
M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 30
SHAPES = [("qkv+stack", 12288, 4096, EPI_NONE, 1536), ("o+stack", 4096, 4096, EPI_RESIDUAL, 512),
          ("gate_up", 22016, 4096, EPI_SILU_MUL, 0), ("down", 4096, 11008, EPI_RESIDUAL, 0),
          ("lm_head", 32000, 4096, EPI_NONE, 0)]


def run(name, N, K, epi, extra, mode):
    os.environ["SLX_GEMM_SK"] = "1" if mode == "sk" else "0"
    a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
    ws = []
    for i in range(3):
        w = (torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16)
        ws.append(ops.pack_weight(w, extra_rows=extra) if extra else ops.pack_weight(w))
    n_out = N // 2 if epi == EPI_SILU_MUL else N
    out_dtype = torch.float32 if name == "lm_head" else torch.bfloat16
    c = torch.empty(M, n_out, device=DEV, dtype=out_dtype)
    r = torch.randn(M, n_out, device=DEV).to(out_dtype) if epi == EPI_RESIDUAL else None
    side = torch.empty(M, extra, device=DEV) if extra else None

    def body():
        for i in range(REPS):
            ops.gemm(a, ws[i % 3], c, epilogue=epi, residual=r, side=side)

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
    us = sorted(ts)[len(ts) // 2]
    wbytes = (N + extra) * K * 2
    return {"gemm": name, "mode": mode, "M": M, "us": round(us, 2),
            "GB/s": round(wbytes / us / 1e3, 1)}


SWEEP = {"qkv+stack": [0, 54, 108, 27], "o+stack": [0, 144, 72, 36], "gate_up": [0, 86, 43, 129],
         "down": [0, 128, 64, 32], "lm_head": [0, 125, 63]}
only = os.environ.get("GEMM_BENCH_ONLY")
for name, N, K, epi, extra in SHAPES:
    if only and name not in only.split(","):
        continue
    print(json.dumps(run(name, N, K, epi, extra, "old")), flush=True)
    for G in (SWEEP[name] if os.environ.get("GEMM_BENCH_SWEEP") else [0]):
        os.environ["SLX_SK_CTAS"] = str(G)
        r = run(name, N, K, epi, extra, "sk")
        r["G"] = G
        print(json.dumps(r), flush=True)
    os.environ.pop("SLX_SK_CTAS", None)
