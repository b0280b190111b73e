"""Decode against BASELINE config 3's adapter pool: Llama-2-13B shape bf16,
128 adapter slots of ranks {8, 16, 64} (seeded) on q,k,v,o, batch 64 at context 128, per-token
adapters uniform over the pool (seed 0).  The pool is far too large to stack into the
projection weights (4 x 128 x 64 rows per layer = 335 MB), so the model takes the gathered
shrink (slx_lora_shrink reads only the batch's adapters) + fused expands.  Reports the CUDA-graph
step time, the same step on the bare backbone, the LoRA marginal and the bytes it moves (the
distinct adapters' A and B rows + the fp32 v), i.e. GB/s against HBM peak.
python tools/bench_decode_pool.py [steps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
B, CTX, N_SLOTS = 64, 128, 128
cfg = LLAMA2_13B
torch.cuda.set_device(0)
ranks = np.random.default_rng(0).choice([8, 16, 64], size=N_SLOTS)
slots = np.random.default_rng(0).integers(0, N_SLOTS, size=B).astype(np.int32)


def run(targets):
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=B, max_ctx=CTX + 1, n_slots=N_SLOTS,
                       max_rank=64, max_tokens=B, lora_targets=targets)
    m.random_backbone(seed=0)
    if targets:
        for a in range(N_SLOTS):
            m.pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
    g = torch.Generator(device=m.device).manual_seed(7)
    for l in range(cfg.layers):
        m.k_cache[l].normal_(generator=g)
        m.v_cache[l].normal_(generator=g)
    seqs = [m.alloc_seq() for _ in range(B)]
    dg = DecodeGraph(m, seqs, slots.tolist() if targets else [-1] * B, fixed_pos=CTX)
    dg.capture()
    for _ in range(5):
        dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dg.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    from paper_2505_14468_b200 import ops
    with ops.KernelTimer() as kt:   # eager step, events around every launch (per class)
        torch.cuda._sleep(200_000_000)
        dg._step()
    torch.cuda.synchronize()
    classes = {k: [round(v[0], 3), v[1]] for k, v in kt.durations().items()}
    info = {"eager_ms_by_class": classes, "decode_lora": m.decode_lora, "stacked_rows_gb": m.memory_ledger()["adapter_stacked_rows"] / 1e9,
            "kernels_per_step": dg.kernels_per_step}
    del dg, m
    torch.cuda.empty_cache()
    return ms, info


ms, info = run(("q", "k", "v", "o"))
ms0, info0 = run(())
d, qd, kvd = cfg.hidden, cfg.q_dim, cfg.kv_dim
distinct = sorted(set(slots.tolist()))
moved = cfg.layers * sum(int(ranks[a]) * (3 * d + qd + qd + 2 * kvd + d) * 2 for a in distinct)
moved += cfg.layers * B * 4 * 64 * 4 * 2   # fp32 v written + read (4 targets, max_rank 64)
hbm = bench.peaks()[0]
lora_ms = ms - ms0
out = {"workload": "13B-shape decode, batch 64, ctx 128, 128 slots r{8,16,64} on q,k,v,o",
       "step_ms": round(ms, 3), "tokens_per_s": round(B / (ms / 1000.0), 1),
       "bare_backbone_step_ms": round(ms0, 3), "lora_marginal_ms": round(lora_ms, 3),
       "distinct_adapters": len(distinct), "lora_bytes_moved_per_step": moved,
       "lora_GB/s": round(moved / (lora_ms / 1000.0) / 1e9, 1) if lora_ms > 0 else None,
       "lora_frac_hbm": round(moved / (lora_ms / 1000.0) / 1e9 / hbm, 4) if lora_ms > 0 else None,
       "floor_ms_at_hbm_peak": round(moved / hbm / 1e6, 3),
       "bare_eager_ms_by_class": info0["eager_ms_by_class"], **info}
print(json.dumps(out))
