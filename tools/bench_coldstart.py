"""Config 5 (BASELINE.json) on one B200: cold-start TTFT of LoRA functions whose artifacts sit in
pinned host memory.  Measures the pre-loader's host->HBM copy of a Llama-2-7B-shape bf16
backbone (13.48 GB incl. embeddings) and of r16 q,k,v,o adapter blobs (32 MiB each), then one
merged prefill of N 512-token prompts (N = concurrent LoRA functions), and prints
TTFT(N) = backbone load + N adapter loads + prefill against the reference's modelled cold start
(sequential sum of container init, library, backbone, adapter and kernel loads,
slorasim engine.py:189-235, profiles.py:39,51).  The NVLink broadcast leg needs >= 2 GPUs
(tests cover its host logic with gloo); this box has one.
python tools/bench_coldstart.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402
from paper_2505_14468_b200.preload import HostArtifactStore, Preloader  # noqa: E402

cfg = LLAMA2_7B
d, f, V, L = cfg.hidden, cfg.ffn, cfg.vocab, cfg.layers
backbone_bytes = 2 * (2 * V * d + L * (4 * d * d + 3 * d * f + 2 * d) + d)
lora = LoraConfig(16, 32.0, ("q", "k", "v", "o"))
adapter_bytes = 2 * L * 4 * lora.rank * 2 * d
N_MAX = 8
t0 = time.time()
store = HostArtifactStore(backbone_bytes + N_MAX * adapter_bytes + (N_MAX + 2) * 4096)
store.put("backbone", np.zeros(backbone_bytes, dtype=np.uint8))
for a in range(N_MAX):
    store.put(f"adapter{a}", np.zeros(adapter_bytes, dtype=np.uint8))
host_setup_s = time.time() - t0
pre = Preloader(store, "cuda")
bb_ms = pre.timed_load_ms("backbone", reps=3)
ad_ms = pre.timed_load_ms("adapter0", reps=5)
# the served model (random init: the copied bytes above stand in for its weights)
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=N_MAX, max_ctx=640, n_slots=N_MAX,
                   max_rank=16, max_tokens=N_MAX * 512)
m.use_stacked_decode = False
m.random_backbone(seed=0)
for a in range(N_MAX):
    m.pool.load_random(a, lora, seed=a)
rng = np.random.default_rng(0)
rows = []
for n in (1, 2, 4, 8):
    prompts = [list(map(int, rng.integers(1, V, size=512))) for _ in range(n)]
    m.prefill(prompts, list(range(n)))   # warm
    for s in list(range(m.max_seqs)):
        if s not in m.free_seqs:
            m.free_seq(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    seqs, _ = m.prefill(prompts, list(range(n)))
    e1.record()
    torch.cuda.synchronize()
    for s in seqs:
        m.free_seq(s)
    pf_ms = e0.elapsed_time(e1)
    ttft = bb_ms + n * ad_ms + pf_ms
    # reference model (profiles.py: 7B backbone cold 7000 ms / from container 280 ms; adapter
    # 100 / 4 ms; prefill T0 + alpha (b - 1) = 500 + 100 (n - 1) ms)
    ref_cold = 7000 + 100 * n + 500 + 100 * (n - 1)
    rows.append({"concurrent_functions": n, "ttft_ms": round(ttft, 2), "prefill_ms": round(pf_ms, 2),
                 "reference_model_cold_ttft_ms": ref_cold})
print(json.dumps({
    "config": "config5: 7B-shape backbone + r16 q,k,v,o adapters from pinned host memory, 1 B200",
    "backbone_bytes": backbone_bytes, "backbone_load_ms": round(bb_ms, 2),
    "backbone_h2d_GBps": round(backbone_bytes / bb_ms / 1e6, 2),
    "adapter_bytes": adapter_bytes, "adapter_load_ms": round(ad_ms, 3),
    "adapter_h2d_GBps": round(adapter_bytes / ad_ms / 1e6, 2),
    "host_store_setup_s": round(host_setup_s, 2), "ttft_vs_concurrency": rows,
    "note": "TTFT = backbone H2D + N adapter H2D + one merged prefill of N x 512 tokens; the "
            "reference column is slorasim's modelled cold start for the same N"}))
store.close()
