"""Config 3 (BASELINE.json): Llama-2-13B-shape bf16 backbone + 128 adapters of mixed rank
{8,16,64} (seeded), prefill of 8 prompts x 2048 tokens per GPU, one adapter per prompt.
Prints bench.run_prefill's JSON (prefill tokens/s, GEMM / attention tensor fractions, kernel
classes, optional bare-backbone LoRA marginal).
python tools/bench_prefill.py [--steps K] [--warmup W] [--no-bare]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--no-bare", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    print(json.dumps(bench.run_prefill(a.steps, a.warmup, bare=not a.no_bare)))
