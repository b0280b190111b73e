"""Generate the config-1 golden fixture with an INDEPENDENT implementation.

Backbone: Hugging Face transformers ``LlamaForCausalLM`` (fp32, CPU, eager
attention) loaded with the seeded init spec's weights.  LoRA: forward hooks on
the q/k/v/o ``nn.Linear`` modules adding ``(alpha/r) (x A^T) B^T`` — the
unmerged formulation of ``/root/reference/PAPER.md:614-621,645-646``.  Greedy
decoding recomputes the full sequence every step (no KV cache), so the fixture
shares no code path with the oracle or the GPU runtime.

Run from the repo root:  python tests/golden/make_golden.py
Writes tests/golden/config1.npz.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2505_14468_b200.config import (  # noqa: E402
    TINY, TINY_LORA, init_adapter, init_backbone, synthetic_requests)

SEED = 0
N_REQ = 16
N_ADAPTERS = 4
N_NEW = 32


def weights_digest(w: dict) -> str:
    h = hashlib.sha256()
    for k in sorted(w):
        h.update(k.encode())
        h.update(np.ascontiguousarray(w[k], np.float32).tobytes())
    return h.hexdigest()


def build_hf(cfg, w):
    from transformers import LlamaConfig, LlamaForCausalLM
    hc = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                     num_hidden_layers=cfg.layers, num_attention_heads=cfg.heads,
                     num_key_value_heads=cfg.kv_heads, head_dim=cfg.head_dim,
                     rms_norm_eps=cfg.rms_eps, rope_theta=cfg.rope_theta,
                     max_position_embeddings=4096, tie_word_embeddings=False,
                     attention_bias=False, mlp_bias=False)
    hc._attn_implementation = "eager"
    m = LlamaForCausalLM(hc).float().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
          "lm_head.weight": w["lm_head"]}
    for i in range(cfg.layers):
        p, q = f"layers.{i}.", f"model.layers.{i}."
        sd[q + "input_layernorm.weight"] = w[p + "input_norm"]
        sd[q + "post_attention_layernorm.weight"] = w[p + "post_norm"]
        sd[q + "self_attn.q_proj.weight"] = w[p + "wq"]
        sd[q + "self_attn.k_proj.weight"] = w[p + "wk"]
        sd[q + "self_attn.v_proj.weight"] = w[p + "wv"]
        sd[q + "self_attn.o_proj.weight"] = w[p + "wo"]
        sd[q + "mlp.gate_proj.weight"] = w[p + "w_gate"]
        sd[q + "mlp.up_proj.weight"] = w[p + "w_up"]
        sd[q + "mlp.down_proj.weight"] = w[p + "w_down"]
    missing, unexpected = m.load_state_dict({k: torch.from_numpy(v) for k, v in sd.items()},
                                            strict=False)
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    return m


class LoraHooks:
    """Per-forward active adapter injected on q/k/v/o/gate/up/down Linear modules."""

    NAMES = {"q": "self_attn.q_proj", "k": "self_attn.k_proj", "v": "self_attn.v_proj",
             "o": "self_attn.o_proj", "gate": "mlp.gate_proj", "up": "mlp.up_proj",
             "down": "mlp.down_proj"}

    def __init__(self, model, cfg, adapters, scale, targets):
        self.active = None
        for i in range(cfg.layers):
            layer = model.model.layers[i]
            for t in targets:
                mod = layer.get_submodule(self.NAMES[t])
                mod.register_forward_hook(self._hook(i, t, adapters, scale))

    def _hook(self, i, t, adapters, scale):
        def fn(_mod, inp, out):
            if self.active is None or self.active < 0:
                return out
            A = torch.from_numpy(adapters[self.active][f"layers.{i}.{t}.A"])
            B = torch.from_numpy(adapters[self.active][f"layers.{i}.{t}.B"])
            return out + scale * ((inp[0] @ A.T) @ B.T)
        return fn


def main():
    torch.manual_seed(0)
    torch.set_num_threads(max(1, len(os.sched_getaffinity(0))))
    cfg, lora = TINY, TINY_LORA
    w = init_backbone(cfg, SEED)
    adapters = [init_adapter(cfg, lora, SEED, a) for a in range(N_ADAPTERS)]
    reqs = synthetic_requests(N_REQ, N_ADAPTERS, cfg.vocab, SEED, max_new_tokens=N_NEW)
    model = build_hf(cfg, w)
    hooks = LoraHooks(model, cfg, adapters, lora.scale, lora.targets)

    toks = np.zeros((N_REQ, N_NEW), np.int64)
    margin = np.zeros((N_REQ, N_NEW), np.float32)
    lse = np.zeros((N_REQ, N_NEW), np.float64)
    lsum = np.zeros((N_REQ, N_NEW), np.float64)
    lsq = np.zeros((N_REQ, N_NEW), np.float64)
    keep = {}
    with torch.no_grad():
        for r, req in enumerate(reqs):
            hooks.active = req.adapter
            seq = list(req.prompt)
            for s in range(N_NEW):
                logits = model(torch.tensor([seq])).logits[0, -1].numpy().astype(np.float32)
                top = np.partition(logits, -2)[-2:]
                margin[r, s] = top[1] - top[0]
                lg = logits.astype(np.float64)
                lse[r, s] = lg.max() + np.log(np.exp(lg - lg.max()).sum())
                lsum[r, s] = lg.sum()
                lsq[r, s] = (lg * lg).sum()
                if r < 4 and s in (0, N_NEW - 1):
                    keep[(r, s)] = logits
                nxt = int(np.argmax(logits))
                toks[r, s] = nxt
                seq.append(nxt)
    prompt_flat = np.concatenate([np.asarray(q.prompt, np.int64) for q in reqs])
    prompt_indptr = np.concatenate([[0], np.cumsum([len(q.prompt) for q in reqs])]).astype(np.int64)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config1.npz")
    np.savez_compressed(
        out, seed=SEED, n_adapters=N_ADAPTERS, n_new=N_NEW,
        prompt_flat=prompt_flat, prompt_indptr=prompt_indptr,
        adapter_ids=np.asarray([q.adapter for q in reqs], np.int64),
        tokens=toks, margin=margin, lse=lse, logit_sum=lsum, logit_sumsq=lsq,
        kept_index=np.asarray(sorted(keep), np.int64),
        kept_logits=np.stack([keep[k] for k in sorted(keep)]),
        weights_sha256=np.asarray(weights_digest(w)),
        generator=np.asarray("transformers-%s torch-%s LlamaForCausalLM eager fp32 + lora hooks"
                             % (__import__("transformers").__version__, torch.__version__)))
    print("wrote", out, "min margin", float(margin.min()))


if __name__ == "__main__":
    main()
