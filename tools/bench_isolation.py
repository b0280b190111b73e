"""Isolation mode at the 7B shape (§8 f3): K function processes over one CUDA-IPC-shared 7B
backbone.  Reports each process's own device bytes and measured CUDA-context bytes (the
reference books 473 MB per process, profiles.py:22), the per-GPU footprint with sharing vs one
private backbone per function (the reference's NBS ablation), and per-function prefill/decode
latency in its own process.  python tools/bench_isolation.py [K]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.isolation import IsolatedFunctions  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    lora = LoraConfig(16, 32.0, ("q", "k", "v", "o"))
    m = MultiLoraModel(LLAMA2_7B, dtype=torch.bfloat16, max_seqs=4, max_ctx=256, n_slots=1,
                       max_rank=16, max_tokens=512)
    m.random_backbone(seed=0)
    torch.cuda.synchronize()
    # adapters travel as host dicts (the function's own artifact)
    m.pool.load_random(0, lora, seed=1)
    blob = m.pool.blobs[0].cpu()
    layout, _ = m.pool.blob_layout(lora.rank)
    ad = {}
    for l, t, ao, bo, di, do in layout:
        ad[f"layers.{l}.{t}.A"] = blob[ao:ao + lora.rank * di].view(lora.rank, di).float().numpy()
        ad[f"layers.{l}.{t}.B"] = blob[bo:bo + do * lora.rank].view(do, lora.rank).float().numpy()
    m.pool.evict(0)
    bb = m.backbone_bytes()
    t0 = time.time()
    iso = IsolatedFunctions(m, {f"f{i}": ad for i in range(K)}, lora, max_seqs=4, max_ctx=256,
                            max_tokens=512)
    start_s = time.time() - t0
    res = {"functions": K, "backbone_bytes": bb, "spawn_all_s": start_s, "per_function": {}}
    prompts = [list(range(1, 61))]
    for fid in iso.info:
        iso.run(fid, prompts, 4)   # warm-up
        t = time.time()
        iso.run(fid, prompts, 33)
        res["per_function"][fid] = {**iso.info[fid], "prefill60_plus_32_decode_s": time.time() - t}
    iso.close()
    ctx = [v["context_bytes"] for v in res["per_function"].values()]
    own = [v["own_bytes"] for v in res["per_function"].values()]
    res["context_bytes_median"] = sorted(ctx)[len(ctx) // 2]
    res["reference_context_overhead_bytes"] = 473_000_000
    res["shared_footprint_bytes"] = bb + sum(own) + sum(ctx)
    res["private_backbones_footprint_bytes"] = K * bb + sum(own) + sum(ctx)
    print(json.dumps(res))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/isolation.json", "w"), indent=1)


if __name__ == "__main__":
    main()
