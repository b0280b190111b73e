"""numpy fp32 restatement of the shared-backbone multi-LoRA forward (TEST INFRA ONLY).

Algorithm sources:
- unmerged LoRA: backbone and adapter computed separately and summed
  (``/root/reference/PAPER.md:614-621``; "unmerged inference atop Transformers",
  ``PAPER.md:645-646``);  y = x W^T + (alpha/r) (x A^T) B^T, PEFT layout.
- backbone: Llama-2 (``PAPER.md:672``) — RMSNorm, rotary embeddings
  (rotate-half convention), causal MHA/GQA, SwiGLU MLP, untied lm_head.
- the batch is the mixed, adapter-segmented batch the runtime forms from the
  batcher's ``FlushDecision``s (``pkg/src/slorasim/batching.py:99-154``):
  prefill is token-major with ``seg_indptr`` (SGMV semantics), decode is one
  token per request with a per-token adapter slot (BGMV semantics).

Everything is float32; matmuls go through numpy's BLAS.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


# --------------------------------------------------------------------------- primitives

def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    x = x.astype(F32, copy=False)
    var = np.mean(x * x, axis=-1, keepdims=True, dtype=F32)
    return (x * (F32(1.0) / np.sqrt(var + F32(eps)))).astype(F32) * w


def rope_table(max_pos: int, head_dim: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_pos, head_dim//2], computed in float64 then rounded to fp32."""
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def apply_rope(x: np.ndarray, pos: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """x [T, H, D]; rotate-half: (x1, x2) -> (x1 c - x2 s, x2 c + x1 s)."""
    half = x.shape[-1] // 2
    c = cos[pos][:, None, :]
    s = sin[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(F32)


def silu(x: np.ndarray) -> np.ndarray:
    return (x / (F32(1.0) + np.exp(-x))).astype(F32)


def lora_delta(x: np.ndarray, A: np.ndarray, B: np.ndarray, scale: float) -> np.ndarray:
    """(alpha/r) (x A^T) B^T for one adapter; x [T, d_in], A [r, d_in], B [d_out, r]."""
    v = x @ A.T
    return (F32(scale) * (v @ B.T)).astype(F32)


def bgmv(y: np.ndarray, x: np.ndarray, A_pool: list, B_pool: list, scales,
         tok_slot: np.ndarray) -> np.ndarray:
    """Decode LoRA: y[t] += s_a (x[t] A_a^T) B_a^T with a = tok_slot[t] (-1 = none)."""
    y = y.copy()
    for a in np.unique(tok_slot):
        if a < 0:
            continue
        rows = np.nonzero(tok_slot == a)[0]
        y[rows] += lora_delta(x[rows], A_pool[a], B_pool[a], scales[a])
    return y


def sgmv(y: np.ndarray, x: np.ndarray, A_pool: list, B_pool: list, scales,
         seg_indptr: np.ndarray, seg_slot: np.ndarray) -> np.ndarray:
    """Prefill LoRA over contiguous segments: tokens [p_s, p_{s+1}) use seg_slot[s]."""
    y = y.copy()
    for s in range(len(seg_slot)):
        a = int(seg_slot[s])
        lo, hi = int(seg_indptr[s]), int(seg_indptr[s + 1])
        if a < 0 or hi <= lo:
            continue
        y[lo:hi] += lora_delta(x[lo:hi], A_pool[a], B_pool[a], scales[a])
    return y


def softmax_rows(s: np.ndarray) -> np.ndarray:
    m = np.max(s, axis=-1, keepdims=True)
    e = np.exp(s - m)
    return (e / np.sum(e, axis=-1, keepdims=True, dtype=F32)).astype(F32)


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, q_pos: np.ndarray) -> np.ndarray:
    """One sequence. q [Tq, H, D]; k, v [Tk, Hkv, D]; query at absolute position
    q_pos[i] attends keys 0..q_pos[i] (causal)."""
    H, D = q.shape[1], q.shape[2]
    Hkv = k.shape[1]
    group = H // Hkv
    out = np.empty_like(q)
    scale = F32(1.0 / np.sqrt(D))
    kpos = np.arange(k.shape[0])
    mask = kpos[None, :] > q_pos[:, None]
    for h in range(H):
        kh = k[:, h // group, :]
        vh = v[:, h // group, :]
        s = (q[:, h, :] @ kh.T) * scale
        s = np.where(mask, F32(-np.inf), s).astype(F32)
        out[:, h, :] = softmax_rows(s) @ vh
    return out


# --------------------------------------------------------------------------- model

class OracleModel:
    """Mixed-batch multi-LoRA Llama forward with per-request KV state.

    ``adapters[a]`` is a dict ``layers.{i}.{t}.A/B`` for adapter slot ``a``;
    ``scales[a]`` = alpha/r of that adapter; a request with adapter ``-1`` uses
    the bare backbone.
    """

    def __init__(self, cfg, weights: dict, adapters: list[dict], scales: list[float],
                 targets: tuple[str, ...], max_pos: int = 4096):
        self.cfg = cfg
        self.w = weights
        self.adapters = adapters
        self.scales = list(scales)
        self.targets = tuple(targets)
        self.cos, self.sin = rope_table(max_pos, cfg.head_dim, cfg.rope_theta)
        self.kv: list[list[tuple[np.ndarray, np.ndarray]]] = []  # per request, per layer

    # -- one projection with the segmented LoRA term
    def _proj(self, layer: int, t: str, x: np.ndarray, W: np.ndarray,
              seg_indptr: np.ndarray, seg_slot: np.ndarray) -> np.ndarray:
        y = (x @ W.T).astype(F32)
        if t in self.targets:
            A = [ad[f"layers.{layer}.{t}.A"] for ad in self.adapters]
            B = [ad[f"layers.{layer}.{t}.B"] for ad in self.adapters]
            y = sgmv(y, x, A, B, self.scales, seg_indptr, seg_slot)
        return y

    def _forward(self, tokens: np.ndarray, positions: np.ndarray, seg_indptr: np.ndarray,
                 seg_slot: np.ndarray, seq_of_seg: list[int]) -> np.ndarray:
        """Token-major forward; every segment s is a contiguous run of sequence
        seq_of_seg[s] continuing at positions[...]. Appends to self.kv."""
        cfg, w = self.cfg, self.w
        H, Hkv, D = cfg.heads, cfg.kv_heads, cfg.head_dim
        x = w["embed"][tokens].astype(F32)
        for i in range(cfg.layers):
            p = f"layers.{i}."
            hn = rmsnorm(x, w[p + "input_norm"], cfg.rms_eps)
            q = self._proj(i, "q", hn, w[p + "wq"], seg_indptr, seg_slot).reshape(-1, H, D)
            k = self._proj(i, "k", hn, w[p + "wk"], seg_indptr, seg_slot).reshape(-1, Hkv, D)
            v = self._proj(i, "v", hn, w[p + "wv"], seg_indptr, seg_slot).reshape(-1, Hkv, D)
            q = apply_rope(q, positions, self.cos, self.sin)
            k = apply_rope(k, positions, self.cos, self.sin)
            attn = np.empty_like(q)
            for s, seq in enumerate(seq_of_seg):
                lo, hi = int(seg_indptr[s]), int(seg_indptr[s + 1])
                kc, vc = self.kv[seq][i]
                kc = np.concatenate([kc, k[lo:hi]], axis=0)
                vc = np.concatenate([vc, v[lo:hi]], axis=0)
                self.kv[seq][i] = (kc, vc)
                attn[lo:hi] = attention(q[lo:hi], kc, vc, positions[lo:hi])
            o = self._proj(i, "o", attn.reshape(-1, H * D), w[p + "wo"], seg_indptr, seg_slot)
            x = (x + o).astype(F32)
            hn = rmsnorm(x, w[p + "post_norm"], cfg.rms_eps)
            g = self._proj(i, "gate", hn, w[p + "w_gate"], seg_indptr, seg_slot)
            u = self._proj(i, "up", hn, w[p + "w_up"], seg_indptr, seg_slot)
            mlp = self._proj(i, "down", (silu(g) * u).astype(F32), w[p + "w_down"],
                             seg_indptr, seg_slot)
            x = (x + mlp).astype(F32)
        return rmsnorm(x, w["final_norm"], cfg.rms_eps)

    def logits(self, h: np.ndarray) -> np.ndarray:
        return (h @ self.w["lm_head"].T).astype(F32)

    def prefill(self, prompts: list[list[int]], adapter_ids: list[int]) -> np.ndarray:
        """Start len(prompts) sequences; returns last-position logits [n, V]."""
        n = len(prompts)
        base = len(self.kv)
        Hkv, D = self.cfg.kv_heads, self.cfg.head_dim
        for _ in range(n):
            self.kv.append([(np.zeros((0, Hkv, D), F32), np.zeros((0, Hkv, D), F32))
                            for _ in range(self.cfg.layers)])
        lens = [len(p) for p in prompts]
        seg_indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tokens = np.concatenate([np.asarray(p, np.int64) for p in prompts])
        positions = np.concatenate([np.arange(L) for L in lens]).astype(np.int64)
        h = self._forward(tokens, positions, seg_indptr, np.asarray(adapter_ids),
                          [base + s for s in range(n)])
        last = seg_indptr[1:] - 1
        return self.logits(h[last])

    def teacher_forced(self, tokens: list[int], adapter_id: int) -> np.ndarray:
        """Logits at every position of one sequence (fresh KV state) [L, V]."""
        self.kv.append([(np.zeros((0, self.cfg.kv_heads, self.cfg.head_dim), F32),
                         np.zeros((0, self.cfg.kv_heads, self.cfg.head_dim), F32))
                        for _ in range(self.cfg.layers)])
        L = len(tokens)
        h = self._forward(np.asarray(tokens, np.int64), np.arange(L), np.array([0, L]),
                          np.array([adapter_id]), [len(self.kv) - 1])
        return self.logits(h)

    def decode(self, seqs: list[int], tokens: list[int], adapter_ids: list[int]) -> np.ndarray:
        """One token for each sequence in ``seqs``; returns logits [n, V]."""
        n = len(seqs)
        positions = np.asarray([self.kv[s][0][0].shape[0] for s in seqs], np.int64)
        seg_indptr = np.arange(n + 1, dtype=np.int64)
        h = self._forward(np.asarray(tokens, np.int64), positions, seg_indptr,
                          np.asarray(adapter_ids), list(seqs))
        return self.logits(h)

    def generate(self, prompts, adapter_ids, n_new: int):
        """Greedy decode. Returns (tokens [n, n_new], logits [n, n_new, V])."""
        logits = self.prefill(prompts, adapter_ids)
        n = len(prompts)
        seqs = list(range(len(self.kv) - n, len(self.kv)))
        toks = np.zeros((n, n_new), np.int64)
        all_logits = np.zeros((n, n_new, self.cfg.vocab), F32)
        for step in range(n_new):
            all_logits[:, step] = logits
            toks[:, step] = np.argmax(logits, axis=-1)
            if step + 1 < n_new:
                logits = self.decode(seqs, list(toks[:, step]), adapter_ids)
        return toks, all_logits


def top2_margin(logits: np.ndarray) -> np.ndarray:
    """top-1 minus top-2 logit along the last axis."""
    part = np.partition(logits, -2, axis=-1)
    return part[..., -1] - part[..., -2]
