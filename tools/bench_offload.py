"""Offload demotion on B200 (§8 f2): measured device -> pinned-host demotion of a 7B r16 adapter
and of the whole 7B backbone through Offloader.apply (slx_offload_d2h), and the promotion of
the adapter back through the pre-loader, vs the reference's modelled demotion at
demotion_gbps = 1 GB/s (engine.py:76, offload.py:219).  python tools/bench_offload.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402
from paper_2505_14468_b200.offload import Eviction, Offloader  # noqa: E402
from paper_2505_14468_b200.preload import HostArtifactStore, Preloader  # noqa: E402
from paper_2505_14468_b200.spec import ArtifactKind  # noqa: E402

m = MultiLoraModel(LLAMA2_7B, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=4, max_rank=16,
                   max_tokens=64)
m.random_backbone(seed=0)
lora = LoraConfig(16, 32.0, ("q", "k", "v", "o"))
for a in range(3):
    m.pool.load_random(a, lora, seed=a)
torch.cuda.synchronize()
ad_bytes = m.pool.blobs[0].numel() * 2
bb_bytes = sum(getattr(t, "data", t).numel() * 2 for t in m.w.values())
store = HostArtifactStore(bb_bytes + 4 * ad_bytes + (64 << 20))
off = Offloader(m, store, {"f0": 0, "f1": 1, "f2": 2}, backbone_fid="llama7b")
res = {"adapter_bytes": ad_bytes, "backbone_bytes": bb_bytes, "reference_demotion_gbps": 1.0}
ad_ms = []
for fid in ("f0", "f1"):
    (ms, _), = off.apply([Eviction(fid, ArtifactKind.ADAPTER_MODEL, "gpu0", ad_bytes, "host0a")])
    ad_ms.append(ms)
res["adapter_demote_ms"] = ad_ms
res["adapter_demote_GBps"] = ad_bytes / (min(ad_ms) / 1e3) / 1e9
pre = Preloader(store, m.device)
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record(pre.copy_stream)
ev = off.promote("f0", pre)
t1.record(pre.copy_stream)
t1.synchronize()
res["adapter_promote_ms"] = t0.elapsed_time(t1)
(ms, _), = off.apply([Eviction("llama7b", ArtifactKind.BACKBONE_MODEL, "gpu0", bb_bytes, "host0a")])
res["backbone_demote_ms"] = ms
res["backbone_demote_GBps"] = bb_bytes / (ms / 1e3) / 1e9
res["reference_model_ms"] = {"adapter": ad_bytes / 1e9 * 1e3, "backbone": bb_bytes / 1e9 * 1e3}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/offload.json", "w"), indent=1)
store.close()
