"""Config 3 (BASELINE.json): Llama-2-13B-shape bf16 backbone + 128 adapters of mixed rank
{8,16,64} (seeded), prefill of 8 prompts x 2048 tokens per GPU, one adapter per prompt.
Prints one JSON line: prefill tokens/s, step time, per-kernel-class device time, the backbone
GEMM tensor-pipe fraction (2*M*N*K over measured GEMM time vs MEASURED_PEAKS bf16 sustained)
and SGMV bytes/s."""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

P, L, N_AD = 8, 2048, 128


def main(steps=3, warmup=1):
    torch.cuda.set_device(0)
    cfg = LLAMA2_13B
    rng = np.random.default_rng(0)
    ranks = rng.choice([8, 16, 64], size=N_AD)
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=P, max_ctx=L, n_slots=N_AD,
                       max_rank=64, max_tokens=P * L)
    m.use_stacked_decode = False
    m.random_backbone(seed=0)
    for a in range(N_AD):
        m.pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
    slots = rng.choice(N_AD, size=P, replace=False)
    dev = m.device
    toks = torch.from_numpy(rng.integers(1, cfg.vocab, size=P * L).astype(np.int32)).to(dev)
    pos = torch.from_numpy(np.tile(np.arange(L, dtype=np.int32), P)).to(dev)
    seq = torch.from_numpy(np.repeat(np.arange(P, dtype=np.int32), L)).to(dev)
    slot = torch.from_numpy(np.repeat(slots.astype(np.int32), L)).to(dev)
    last = torch.from_numpy((np.arange(P) + 1) * L - 1).to(dev)
    segs = [(i * L, L, i, 0) for i in range(P)]
    step = lambda: m.forward(toks, pos, seq, slot, last, segments=segs)  # noqa: E731
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    with ops.KernelTimer() as kt:
        torch.cuda._sleep(200_000_000)
        step()
    torch.cuda.synchronize()
    dur = {k: (round(v[0], 3), v[1]) for k, v in kt.durations().items()}
    T = P * L
    d, f, qd, kvd = cfg.hidden, cfg.ffn, cfg.q_dim, cfg.kv_dim
    gemm_flops = 2 * T * cfg.layers * d * (qd + 2 * kvd + qd + 3 * f)   # lm_head only on P rows
    gemm_flops += 2 * P * d * cfg.vocab
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    tf_peak = float(peaks.get("bf16_tflops_sustained", 1382.1))
    g_ms = kt.durations()["gemm"][0]
    tflops = gemm_flops / (g_ms / 1000.0) / 1e12
    lora_bytes = 0
    for t in ("q", "k", "v", "o"):
        di, do = cfg.target_dims(t)
        lora_bytes += sum(int(ranks[s]) * (di + do) * 2 for s in slots) + T * di * 2 + 2 * T * do * 2
    lora_bytes *= cfg.layers
    l_ms = kt.durations().get("lora", (0.0,))[0]
    # LoRA marginal: the same prefill on the bare backbone (same weights, no LoRA targets)
    del m
    torch.cuda.empty_cache()
    m0 = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=P, max_ctx=L, n_slots=N_AD,
                        max_rank=64, max_tokens=P * L, lora_targets=())
    m0.random_backbone(seed=0)
    step0 = lambda: m0.forward(toks, pos, seq, slot, last, segments=segs)  # noqa: E731
    for _ in range(warmup):
        step0()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        step0()
    e1.record()
    torch.cuda.synchronize()
    ms0 = e0.elapsed_time(e1) / steps
    print(json.dumps({
        "config": "config3: llama2-13b-shape bf16 prefill, 8 x 2048 tokens, 128 adapters r{8,16,64} (q,k,v,o)",
        "prefill_ms": round(ms, 2), "prefill_tokens_per_s": round(T / (ms / 1000.0), 1),
        "ttft_ms_8x2048": round(ms, 2),
        "gemm": {"ms": round(g_ms, 2), "TFLOP/s": round(tflops, 1), "peak": tf_peak,
                 "frac": round(tflops / tf_peak, 4), "flops": gemm_flops},
        "lora": {"marginal_ms": round(ms - ms0, 2), "backbone_only_prefill_ms": round(ms0, 2),
                 "GB/s": round(lora_bytes / ((ms - ms0) / 1000.0) / 1e9, 1) if ms > ms0 else None,
                 "bytes": lora_bytes, "shrink_kernels_ms": round(l_ms, 2),
                 "method": "prefill time minus the same prefill on the bare backbone; the expand "
                           "is an extra K block of the backbone qkv/o GEMMs, the shrink a grouped "
                           "tcgen05 GEMM"},
        "kernels_ms": dur, "adapter_ranks_of_batch": [int(ranks[s]) for s in slots],
    }))


if __name__ == "__main__":
    main()
