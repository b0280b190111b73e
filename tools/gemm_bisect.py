"""Bisect the decode GEMM mainloop cost: normal / no X reload / no MMA / neither."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from microbench import timeit  # noqa: E402

for (N, K, name) in [(32000, 4096, "lm_head"), (4096, 4096, "o"), (12288, 4096, "qkv")]:
    a = torch.randn(64, K, device="cuda").to(torch.bfloat16)
    w = ops.pack_weight((torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16))
    for cfg in [dict(), dict(SLX_GEMM_SPLITS="8", SLX_GEMM_CTAS="2")]:
        for dbg in ["0", "1", "2", "3"]:
            os.environ.update(cfg)
            os.environ["SLX_GEMM_DBG"] = dbg
            ms = timeit(lambda: ops.gemm(a, w))
            print(name, cfg, "dbg", dbg, f"{ms*1000:.1f} us", f"{N*K*2/ms/1e6:.0f} GB/s", flush=True)
            for k in cfg:
                del os.environ[k]
    os.environ["SLX_GEMM_DBG"] = "0"
