"""In-graph attribution of the decode step: time the captured step with one kernel class
replaced by a no-op (its marginal cost).  python tools/step_attrib.py [steps] [rounds]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_14468_b200 import ops  # noqa: E402
from paper_2505_14468_b200._lib import load  # noqa: E402
from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig  # noqa: E402
from paper_2505_14468_b200.engine import DecodeGraph  # noqa: E402
from paper_2505_14468_b200.model import MultiLoraModel  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
load()
cfg = LLAMA2_7B
lora = LoraConfig(bench.RANK, bench.ALPHA, ("q", "k", "v", "o"))
m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=bench.BATCH, max_ctx=bench.CTX + 1,
                   n_slots=bench.N_ADAPTERS, max_rank=bench.RANK, max_tokens=bench.BATCH)
m.random_backbone(seed=0)
for a in range(bench.N_ADAPTERS):
    m.pool.load_random(a, lora, seed=1000 + a)
g = torch.Generator(device=m.device).manual_seed(7)
for l in range(cfg.layers):
    m.k_cache[l].normal_(generator=g)
    m.v_cache[l].normal_(generator=g)
seqs = [m.alloc_seq() for _ in range(bench.BATCH)]
slots = bench.tok_slots().tolist()
orig = {k: getattr(ops, k) for k in ("gemm", "rope_attention_decode", "rmsnorm", "rmsnorm_lora")}


def gemm_kind(w):
    n, k = w.shape
    return {12288: "qkv", 22016: "gate_up", 32000: "lm_head"}.get(n, "o" if k == 4096 else "down")


def patched(skip):
    def gemm(a, w, out=None, **kw):
        if gemm_kind(w) in skip:
            if out is None:
                out = torch.zeros(a.shape[0], w.shape[0], device=a.device,
                                  dtype=kw.get("out_dtype") or torch.bfloat16)
            return out
        return orig["gemm"](a, w, out, **kw)

    def attn(*a, **kw):
        return None if "attn" in skip else orig["rope_attention_decode"](*a, **kw)

    def norm(*a, **kw):
        return None if "norm" in skip else orig["rmsnorm"](*a, **kw)

    def norm_l(*a, **kw):
        if "norm_lora" in skip:
            return None
        return orig["rmsnorm_lora"](*a, **kw)
    return {"gemm": gemm, "rope_attention_decode": attn, "rmsnorm": norm, "rmsnorm_lora": norm_l}


def capture(skip, slot_list):
    for k, f in patched(skip).items():
        setattr(ops, k, f)
    dg = DecodeGraph(m, seqs, slot_list, fixed_pos=bench.CTX)
    dg.capture()
    for k, f in orig.items():
        setattr(ops, k, f)
    return dg


def time_graph(dg):
    for _ in range(2):
        dg.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        dg.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


variants = [("full step", set(), slots), ("no adapters", set(), [-1] * bench.BATCH),
            ("- attention", {"attn"}, slots), ("- rmsnorm (pre-qkv)", {"norm"}, slots),
            ("- rmsnorm_lora (post-attn)", {"norm_lora"}, slots), ("- qkv gemm", {"qkv"}, slots),
            ("- o gemm", {"o"}, slots), ("- gate_up gemm", {"gate_up"}, slots),
            ("- down gemm", {"down"}, slots), ("- lm_head", {"lm_head"}, slots),
            ("- all gemms", {"qkv", "o", "gate_up", "down", "lm_head"}, slots)]
graphs = [(n, capture(s, sl)) for n, s, sl in variants]
res = {n: [] for n, _ in graphs}
for _ in range(rounds):
    for n, dg in graphs:
        res[n].append(time_graph(dg))
base = min(res["full step"])
for n, _ in graphs:
    t = min(res[n])
    print(f"{n:30s} {t:7.3f} ms   marginal {base - t:+7.3f} ms", flush=True)
