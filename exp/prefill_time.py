"""Experiment harness (not product): config-3 prefill step (bench.run_prefill) from a given
libslora_b200 build.  python exp/prefill_time.py [lib.so]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
r = bench.run_prefill(steps=3, warmup=1, bare=False, e2e=False)
print(os.path.basename(_lib.LIB_PATH), json.dumps({"prefill_ms": r["prefill_ms"], "gemm": r["gemm"]["ms"],
                                                  "gemm_frac": r["gemm"]["frac"], "attn": r["attention"]["ms"],
                                                  "kernels_ms": r["kernels_ms"]}))
