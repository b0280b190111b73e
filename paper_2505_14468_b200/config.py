"""Backbone / adapter shapes and the seeded init spec.

The reference has no tensors: its forward is the latency law
``T0 + alpha*(b-1)`` (reference ``pkg/src/slorasim/batching.py:17-21``) and the
backbone is a byte count (``pkg/src/slorasim/profiles.py:30-40,89-99``).  The
shapes below are the public Llama-2 configs the paper serves
(``PAPER.md:672``); the tiny shape is BASELINE.json config 1.

LoRA convention (PEFT layout, unmerged, ``PAPER.md:614-621,645-646``):
``y = x W^T + (alpha/r) * (x A^T) B^T`` with ``A [r, d_in]`` and ``B [d_out, r]``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# LoRA target projections, in the order the runtime lays out adapter pools.
ATTN_TARGETS = ("q", "k", "v", "o")
ALL_TARGETS = ("q", "k", "v", "o", "gate", "up", "down")


@dataclass(frozen=True)
class BackboneConfig:
    name: str
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def q_dim(self) -> int:
        return self.heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    def target_dims(self, target: str) -> tuple[int, int]:
        """(d_in, d_out) of a LoRA target projection."""
        d, f = self.hidden, self.ffn
        return {
            "q": (d, self.q_dim),
            "k": (d, self.kv_dim),
            "v": (d, self.kv_dim),
            "o": (self.q_dim, d),
            "gate": (d, f),
            "up": (d, f),
            "down": (f, d),
        }[target]

    def param_count(self) -> int:
        d, f, v = self.hidden, self.ffn, self.vocab
        per_layer = d * (self.q_dim + 2 * self.kv_dim) + self.q_dim * d + 3 * d * f + 2 * d
        return v * d * 2 + self.layers * per_layer + d

    def linear_weight_bytes_per_step(self) -> int:
        """bf16 bytes of every projection read once by a decode step (lm_head included)."""
        d, f = self.hidden, self.ffn
        per_layer = d * (self.q_dim + 2 * self.kv_dim) + self.q_dim * d + 3 * d * f
        return 2 * (self.layers * per_layer + self.vocab * d)

    def kv_bytes_per_token(self) -> int:
        return 2 * 2 * self.layers * self.kv_dim  # K and V, bf16


TINY = BackboneConfig("tiny", hidden=256, layers=2, heads=4, kv_heads=4, head_dim=64,
                      ffn=688, vocab=32000)
LLAMA2_7B = BackboneConfig("llama2-7b", hidden=4096, layers=32, heads=32, kv_heads=32,
                           head_dim=128, ffn=11008, vocab=32000)
LLAMA2_13B = BackboneConfig("llama2-13b", hidden=5120, layers=40, heads=40, kv_heads=40,
                            head_dim=128, ffn=13824, vocab=32000)
SHAPES = {c.name: c for c in (TINY, LLAMA2_7B, LLAMA2_13B)}


@dataclass(frozen=True)
class LoraConfig:
    """One adapter: rank, alpha and the projections it targets."""

    rank: int
    alpha: float
    targets: tuple[str, ...] = ATTN_TARGETS

    @property
    def scale(self) -> float:
        return self.alpha / self.rank

    def bytes(self, cfg: BackboneConfig, dtype_bytes: int = 2) -> int:
        n = 0
        for t in self.targets:
            di, do = cfg.target_dims(t)
            n += self.rank * (di + do)
        return n * cfg.layers * dtype_bytes


# ---------------------------------------------------------------------------
# Seeded init spec (numpy, platform independent: PCG64 streams keyed by name)
# ---------------------------------------------------------------------------

def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (exactly representable)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    nan = np.isnan(x)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def _rng(seed: int, *key) -> np.random.Generator:
    # Stable named streams: hash the key path into the seed sequence.
    material = [seed] + [sum((i + 1) * ord(c) for i, c in enumerate(str(k))) for k in key]
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(material)))


def init_backbone(cfg: BackboneConfig, seed: int, std: float = 0.02) -> dict[str, np.ndarray]:
    """Random-init backbone, every tensor bf16-representable fp32.

    Norm weights are drawn around 1 (not exactly 1) so a dropped norm weight is
    caught by parity tests.
    """
    w: dict[str, np.ndarray] = {}

    def normal(name, shape, s=std, mean=0.0):
        w[name] = round_to_bf16(mean + s * _rng(seed, name).standard_normal(shape, dtype=np.float32))

    d = cfg.hidden
    normal("embed", (cfg.vocab, d), s=1.0)
    for i in range(cfg.layers):
        p = f"layers.{i}."
        normal(p + "input_norm", (d,), s=0.1, mean=1.0)
        normal(p + "wq", (cfg.q_dim, d))
        normal(p + "wk", (cfg.kv_dim, d))
        normal(p + "wv", (cfg.kv_dim, d))
        normal(p + "wo", (d, cfg.q_dim))
        normal(p + "post_norm", (d,), s=0.1, mean=1.0)
        normal(p + "w_gate", (cfg.ffn, d))
        normal(p + "w_up", (cfg.ffn, d))
        normal(p + "w_down", (d, cfg.ffn))
    normal("final_norm", (d,), s=0.1, mean=1.0)
    normal("lm_head", (cfg.vocab, d))
    return w


def init_adapter(cfg: BackboneConfig, lora: LoraConfig, seed: int, adapter_id: int,
                 std: float = 0.02) -> dict[str, np.ndarray]:
    """Random-init adapter with NON-zero B (PEFT zero-init would test nothing).

    A ~ N(0, 1/d_in) (the scale of PEFT's kaiming init for A), B ~ N(0, std):
    the LoRA term is a sizeable fraction of the projection, so a dropped or
    mis-gathered adapter changes greedy tokens.
    """
    w: dict[str, np.ndarray] = {}
    for i in range(cfg.layers):
        for t in lora.targets:
            di, do = cfg.target_dims(t)
            key = f"adapter{adapter_id}.layers.{i}.{t}"
            w[f"layers.{i}.{t}.A"] = round_to_bf16(
                _rng(seed, key, "A").standard_normal((lora.rank, di), dtype=np.float32)
                / np.float32(np.sqrt(di)))
            w[f"layers.{i}.{t}.B"] = round_to_bf16(
                _rng(seed, key, "B").standard_normal((do, lora.rank), dtype=np.float32) * std)
    return w


@dataclass
class RequestSpec:
    """A synthetic request: prompt token ids and the adapter it carries (-1 = none)."""

    prompt: list[int]
    adapter: int
    max_new_tokens: int = 32


def synthetic_requests(n: int, n_adapters: int, vocab: int, seed: int,
                       min_len: int = 4, max_len: int = 24, max_new_tokens: int = 32,
                       ) -> list[RequestSpec]:
    """Config-1 workload: adapter ``i % n_adapters``, seeded ragged prompt lengths."""
    rng = _rng(seed, "requests")
    out = []
    for i in range(n):
        length = int(rng.integers(min_len, max_len + 1))
        prompt = [int(t) for t in rng.integers(1, vocab, size=length)]
        out.append(RequestSpec(prompt, i % n_adapters if n_adapters > 0 else -1, max_new_tokens))
    return out


TINY_LORA = LoraConfig(rank=8, alpha=16.0, targets=ATTN_TARGETS)
