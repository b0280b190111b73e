"""Real-hardware serving replay (BASELINE metric "p50 TTFT"): a trace made by
the reference's own generator (tools/make_trace.py -> profiles/r02_trace_*.csv) replayed in real
time through ServingRuntime on one B200 — contention-aware batcher rounds, dispatch admission
(KV slots, adapter cold loads from the pinned container tier through the pre-loader, demotion
of idle adapters by the offloader when the adapter pool is full), merged mixed-adapter
prefill, CUDA-graph decode buckets.  Reports the reference's metrics (nearest-rank TTFT /
TPOT / E2E percentiles, output tokens/s, metrics.py:17-25,114-147) and writes the request CSV
in the reference's format.
python tools/serve_trace.py TRACE.csv OUT_PREFIX [resident_slots] [time_scale] [max_sequences]
                            [7b|13b] [r16|mixed] [mix|sep]
(mix (default): decode tokens ride in the round's prefill forward; sep: separate prefill and
decode forwards, ServingRuntime(mixed_rounds=False).
13b mixed: Llama-2-13B shape, each function's adapter rank drawn from {8, 16, 64} -- BASELINE
config 4's 13B family; the adapter pool then exceeds the stacked-decode budget and decode takes
the gathered LoRA kernels.)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14468_b200 import wire  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LLAMA2_13B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402
from paper_2505_14468_b200.offload import Offloader  # noqa: E402
from paper_2505_14468_b200.preload import HostArtifactStore, Preloader  # noqa: E402
from paper_2505_14468_b200.runtime import ServingRuntime  # noqa: E402
from paper_2505_14468_b200.spec import ArtifactKind, ArtifactSpec, FunctionSpec  # noqa: E402

trace_path, out_prefix = sys.argv[1], sys.argv[2]
n_slots = int(sys.argv[3]) if len(sys.argv) > 3 else 24
time_scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
MAX_SEQS = int(sys.argv[5]) if len(sys.argv) > 5 else 128   # concurrent sequences (decode batch)
BACKBONE = sys.argv[6] if len(sys.argv) > 6 else "7b"
RANKS = sys.argv[7] if len(sys.argv) > 7 else "r16"
MIXED_ROUNDS = not (len(sys.argv) > 8 and sys.argv[8] == "sep")
MAX_CTX = 512
torch.cuda.set_device(0)
recs = wire.read_trace_csv(trace_path)
fids = sorted({r.function_id for r in recs})
cfg = LLAMA2_13B if BACKBONE == "13b" else LLAMA2_7B
if RANKS == "mixed":
    rk = np.random.default_rng(0).choice([8, 16, 64], size=len(fids))
    lora_of = {f: LoraConfig(int(r), 2.0 * int(r)) for f, r in zip(fids, rk)}
else:
    lora_of = {f: LoraConfig(16, 32.0) for f in fids}
RANK = max(lo.rank for lo in lora_of.values())
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=MAX_SEQS + 1, max_ctx=MAX_CTX,
                   n_slots=n_slots, max_rank=RANK, max_tokens=4096)
m.random_backbone(seed=0)
# every function's adapter lives in the pinned container tier; the first n_slots are resident
blob_of = {f: m.pool.blob_layout(lora_of[f].rank)[1] * 2 for f in fids}
store = HostArtifactStore(sum(blob_of.values()) * 2 + (64 << 20))
g = torch.Generator(device=m.device).manual_seed(5)
for i, f in enumerate(fids):
    blob = (torch.randn(blob_of[f] // 2, generator=g, device=m.device) * 0.02).to(torch.bfloat16)
    store.put(f"adapter/{f}", blob.cpu())
pre = Preloader(store, m.device)
slot_of = {}
for i, f in enumerate(fids[:n_slots]):
    dev, ev = pre.load(f"adapter/{f}")
    ev.synchronize()
    m.pool.install(i, dev.view(torch.bfloat16), lora_of[f])
    slot_of[f] = i
torch.cuda.synchronize()
# B200-calibrated latency law of the function's backbone (profiles/r02_calibrated_specs.json)
# and the KV reservation the pool really makes per request (max_ctx positions)
cal = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "profiles", "r02_calibrated_specs.json")))
c = cal["functions"]["llama13b" if BACKBONE == "13b" else "llama7b"]
t0 = float(c["prefill_base_ms"])
alpha = float(c["prefill_marginal_ms"])
dec = float(c["decode_ms_per_token_b1"])
kv_req = cfg.kv_bytes_per_token() * MAX_CTX
funcs = {}
for f in fids:
    spec = FunctionSpec(f, (ArtifactSpec(ArtifactKind.ADAPTER_MODEL, blob_of[f], 1.0, 1.0),),
                        5.0 * t0, t0, alpha, dec, kv_req, 0.0, backbone_id=cfg.name)
    funcs[f] = (spec, slot_of.get(f, -1))
adapters = {f: (f"adapter/{f}", lora_of[f]) for f in fids}
off = Offloader(m, store, dict(slot_of))
rt = ServingRuntime(m, funcs, store=store, adapters=adapters, preloader=pre, offloader=off,
                    mixed_rounds=MIXED_ROUNDS)
rt.graphs.warm()
t_start = time.perf_counter()
done = wire.replay(rt, recs, cfg.vocab, seed=0, time_scale=time_scale, max_ctx=MAX_CTX)
wall = time.perf_counter() - t_start
rep = rt.report()
rep.update({"trace": os.path.basename(trace_path), "requests_in_trace": len(recs),
            "functions": len(fids), "resident_adapter_slots": n_slots, "time_scale": time_scale,
            "max_concurrent_sequences": MAX_SEQS,
            "wall_s": round(wall, 2), "cold_loads": sum(1 for v in rt.cold_ms.values() if v),
            "demotions_in_container_tier": len(off.demoted),
            "model": f"{cfg.name} shape bf16, random init; adapters on q,k,v,o of rank "
                     f"{'8/16/64 (seeded per function)' if RANKS == 'mixed' else '16'}",
            "decode_lora": m.decode_lora, "mixed_rounds": MIXED_ROUNDS,
            "slo_ttft_ms": 5.0 * t0})
rep["slo_attainment"] = float(np.mean([(r.first_token_ms - r.arrival_ms) <= 5.0 * t0 for r in done]))
wire.write_requests_csv(sorted(done, key=lambda r: r.request_id), out_prefix + "_requests.csv",
                        rt.cold_ms)
json.dump(rep, open(out_prefix + "_report.json", "w"), indent=1)
print(json.dumps(rep))
