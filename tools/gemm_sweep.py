"""Sweep the decode (swap-AB) GEMM tiling on B200: nsub x CTAs/SM x cluster splits.
Prints the best configuration per shape.  python tools/gemm_sweep.py [M]"""

import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200._lib import EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL  # noqa: E402

DEV = "cuda"
flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)


def timeit(fn, iters=15):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    shapes = [("qkv", 13824, 4096, EPI_NONE), ("o", 4608, 4096, EPI_RESIDUAL),
              ("gate_up", 22016, 4096, EPI_SILU_MUL), ("down", 4096, 11008, EPI_RESIDUAL),
              ("lm_head", 32000, 4096, EPI_NONE)]
    best = {}
    for k in ("SLX_GEMM_CTAS", "SLX_GEMM_SPLITS", "SLX_GEMM_BN"):
        os.environ.pop(k, None)
    for name, N, K, epi in shapes:   # planner's own choice first
        a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
        w = ops.pack_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
        c = torch.empty(M, N // 2 if epi == EPI_SILU_MUL else N, device=DEV, dtype=torch.bfloat16)
        r = torch.randn(M, N, device=DEV).to(torch.bfloat16) if epi == EPI_RESIDUAL else None
        ms = timeit(lambda: ops.gemm(a, w, c, epilogue=epi, residual=r))
        print(json.dumps({"gemm": name, "planner": True, "us": round(ms * 1000, 2),
                          "GB/s": round(N * K * 2 / ms / 1e6, 1)}), flush=True)
    for name, N, K, epi in shapes:
        a = torch.randn(M, K, device=DEV).to(torch.bfloat16)
        w = ops.pack_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
        nout = N // 2 if epi == EPI_SILU_MUL else N
        c = torch.empty(M, nout, device=DEV, dtype=torch.bfloat16)
        r = torch.randn(M, N, device=DEV).to(torch.bfloat16) if epi == EPI_RESIDUAL else None
        ref = None
        byts = N * K * 2
        for bn, ctas, splits in itertools.product([256, 128], [1, 2], [1, 2, 3, 4, 5, 6, 8]):
            if epi == EPI_SILU_MUL and bn == 128:
                continue
            os.environ.update(SLX_GEMM_CTAS=str(ctas), SLX_GEMM_SPLITS=str(splits),
                              SLX_GEMM_BN=str(bn))
            try:
                ms = timeit(lambda: ops.gemm(a, w, c, epilogue=epi, residual=r))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"gemm": name, "ctas": ctas, "splits": splits,
                                  "error": str(e)[:80]}))
                continue
            out = c.float()
            if ref is None:
                ref = out.clone()
            ok = torch.allclose(out, ref, rtol=2e-2, atol=2e-2)
            gbs = byts / ms / 1e6
            rec = {"gemm": name, "bn": bn, "ctas": ctas, "splits": splits,
                   "us": round(ms * 1000, 2), "GB/s": round(gbs, 1), "ok": ok}
            print(json.dumps(rec), flush=True)
            if ok and (name not in best or gbs > best[name]["GB/s"]):
                best[name] = rec
    for k in os.environ.copy():
        if k.startswith("SLX_GEMM_"):
            del os.environ[k]
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
