"""Experiment (not product): host launch time vs device time of a small merged prefill (7B,
4 segments of 64 tokens, 4 r16 adapters, LoRA fold path) -- is the serving prefill host-bound?"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

torch.cuda.set_device(0)
cfg = LLAMA2_7B
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=64, max_ctx=512, n_slots=24, max_rank=16,
                   max_tokens=4096)
m.random_backbone(seed=0)
for a in range(24):
    m.pool.load_random(a, LoraConfig(16, 32.0), seed=100 + a)
rng = np.random.default_rng(0)
cases = [(4, 64, "stacked"), (4, 64, "gather"), (8, 60, "stacked"), (8, 60, "gather"), (2, 200, True),
         (2, 200, "stacked"), (4, 128, True), (4, 128, "stacked"), (16, 64, "stacked"), (16, 64, "gather")]
for nseg, L, fold in cases:
    m.lora_fold = fold is True
    m.prefill_small_lora = fold if isinstance(fold, str) else "stacked"
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=L))) for _ in range(nseg)]
    ids = list(range(nseg))
    for _ in range(3):
        seqs, lg = m.prefill(prompts, ids)
        for s_ in seqs:
            m.free_seq(s_)
    torch.cuda.synchronize()
    host, dev = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        seqs, lg = m.prefill(prompts, ids)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        host.append((t1 - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
        for s_ in seqs:
            m.free_seq(s_)
    n0 = ops.launch_count()
    seqs, lg = m.prefill(prompts, ids)
    for s_ in seqs:
        m.free_seq(s_)
    print(f"{nseg} x {L} tokens (fold {fold}): host launch {np.median(host):.2f} ms, device {np.median(dev):.2f} ms, "
          f"{ops.launch_count() - n0} launches")
for nseg, L, fold in cases:
    m.lora_fold = fold is True
    m.prefill_small_lora = fold if isinstance(fold, str) else "stacked"
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=L))) for _ in range(nseg)]
    with ops.KernelTimer() as kt:
        torch.cuda._sleep(100_000_000)
        seqs, lg = m.prefill(prompts, list(range(nseg)))
    torch.cuda.synchronize()
    for s_ in seqs:
        m.free_seq(s_)
    print(nseg, L, fold, {k: (round(v[0], 2), v[1]) for k, v in kt.durations().items()})
