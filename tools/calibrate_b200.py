"""Calibration bridge (§8 f1 / row a1): measure the reference's per-function latency law on this
B200 with the real kernels — T0 and alpha of predict_ttft(b) = T0 + alpha (b - 1) over mixed
prefills of b 60-token prompts (the reference trace's median prompt), decode ms/token of a
batch-1 step, KV bytes per request, and the pre-loader's host->HBM artifact loads — for the
Llama-2-7B and -13B shapes, r16 adapters on q,k,v,o.  Writes gpurun_out/calibrated_specs.json
(committed as profiles/r0N_calibrated_specs.json, consumed by tools/run_config4.py --cal, which
runs the unchanged reference simulator).
python tools/calibrate_b200.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.calibrate import profile_function_spec  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402
from paper_2505_14468_b200.preload import HostArtifactStore, Preloader  # noqa: E402

out = {"device": torch.cuda.get_device_name(0), "functions": {}}
lora = LoraConfig(16, 32.0, ("q", "k", "v", "o"))
for name, cfg in (("llama7b", LLAMA2_7B), ("llama13b", LLAMA2_13B)):
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=16, max_ctx=128, n_slots=2,
                       max_rank=16, max_tokens=16 * 64)
    m.random_backbone(seed=0)
    m.pool.load_random(0, lora, seed=1)
    spec, raw = profile_function_spec(m, f"{name}-lora", 0, backbone_id=name, prompt_len=60,
                                      batch_sizes=(1, 2, 4, 8, 16))
    # decode step of a full 16-sequence merged batch (the runtime advances all together)
    from paper_2505_14468_b200.calibrate import measure_decode_ms
    dec16 = measure_decode_ms(m, 0, 16, 60)
    bb_bytes = m.backbone_bytes()
    ad_bytes = m.pool.resident_bytes()
    del m
    torch.cuda.empty_cache()
    # artifact loads through the pre-loader (pinned host -> HBM); 256 MB probe, bandwidth scaled
    store = HostArtifactStore(256 << 20)
    store.put("probe", np.zeros(256 << 20, dtype=np.uint8))
    pre = Preloader(store, "cuda")
    probe_ms = pre.timed_load_ms("probe", reps=5)
    gbps = (256 << 20) / probe_ms / 1e6
    store.close()
    out["functions"][name] = {
        "prefill_base_ms": spec.prefill_base_ms, "prefill_marginal_ms": spec.prefill_marginal_ms,
        "decode_ms_per_token_b1": spec.decode_ms_per_token, "decode_step_ms_b16": dec16,
        "kv_bytes_per_request": spec.kv_cache_bytes_per_request,
        "slo_ttft_ms": spec.slo_ttft_ms, "prefill_ms_by_batch": dict(zip(raw["batch_sizes"], raw["prefill_ms"])),
        "backbone_bytes": bb_bytes, "adapter_bytes": ad_bytes, "h2d_GBps": gbps,
        "backbone_load_ms": bb_bytes / gbps / 1e6, "adapter_load_ms": ad_bytes / gbps / 1e6,
    }
    print(name, json.dumps(out["functions"][name]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/calibrated_specs.json", "w"), indent=1)
