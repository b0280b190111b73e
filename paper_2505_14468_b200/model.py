"""Shared-backbone multi-LoRA Llama runtime on one B200.

One resident backbone per GPU (the reference's one-backbone-per-GPU ledger rule,
``/root/reference/pkg/src/slorasim/ledger.py:130-134``) serves a mixed batch whose
tokens each carry an adapter slot; the adapters live in an HBM slot pool.  The
forward is the unmerged LoRA of ``PAPER.md:614-621``: every targeted projection is
``x W^T`` (tcgen05 GEMM) plus ``scale * (x A^T) B^T`` (LoRA shrink/expand kernels)
added into the GEMM output.

Two activation modes share the same packed bf16 weights:
  * ``torch.bfloat16`` — throughput mode (tcgen05 GEMMs, bf16 activations);
  * ``torch.float32``  — parity mode (fp32 activations, fp32 accumulate, bf16 weights
    upcast exactly), used for the bit-exact greedy-token check against the oracle.
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch

from . import _lib, ops
from ._lib import EPI_RESIDUAL, EPI_SILU_MUL
from .config import ATTN_TARGETS, BackboneConfig, LoraConfig


def resolve_device(device) -> torch.device:
    d = torch.device(device)
    if d.type == "cuda" and d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _to_dev(a, device, dtype=torch.bfloat16) -> torch.Tensor:
    t = torch.as_tensor(a) if not isinstance(a, torch.Tensor) else a
    return t.to(device=device, dtype=dtype).contiguous()


def rope_tables(max_pos: int, head_dim: int, theta: float):
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


class AdapterPool:
    """HBM adapter slots.  Slot s holds one adapter as ONE contiguous bf16 blob with
    A_t [r, d_in] and B_t [d_out, r] for every (layer, target), so a single pinned
    H2D copy (or NCCL broadcast) materialises it; device pointer tables
    ``a_ptr[layer][target]`` / ``b_ptr[layer][target]`` (int64 [n_slots]) index it."""

    def __init__(self, cfg: BackboneConfig, targets, n_slots: int, max_rank: int, device):
        self.cfg, self.targets = cfg, tuple(targets)
        self.n_slots, self.max_rank = n_slots, max_rank
        self.device = resolve_device(device)
        L, nt = cfg.layers, len(self.targets)
        self.a_ptr = torch.zeros((L, nt, n_slots), dtype=torch.int64, device=self.device)
        self.b_ptr = torch.zeros((L, nt, n_slots), dtype=torch.int64, device=self.device)
        self.rank = torch.zeros(n_slots, dtype=torch.int32, device=self.device)
        self.scale = torch.zeros(n_slots, dtype=torch.float32, device=self.device)
        self.blobs: list[torch.Tensor | None] = [None] * n_slots
        self.configs: list[LoraConfig | None] = [None] * n_slots
        self._off_cache: dict = {}
        self.on_install = None   # model hooks (stacked-A rows of the projection GEMMs)
        self.on_evict = None

    def blob_layout(self, rank: int):
        """[(layer, target, a_off, b_off, d_in, d_out)] in elements, and total elements."""
        out, off = [], 0
        for l in range(self.cfg.layers):
            for t in self.targets:
                di, do = self.cfg.target_dims(t)
                out.append((l, t, off, off + rank * di, di, do))
                off += rank * (di + do)
        return out, off

    def offsets(self, rank: int, layer: int, target: str) -> tuple[int, int]:
        """Element offsets of A and B of (layer, target) inside a rank-``rank`` blob."""
        key = (rank, layer, target)
        if key not in self._off_cache:
            layout, _ = self.blob_layout(rank)
            for l, t, ao, bo, _di, _do in layout:
                self._off_cache[(rank, l, t)] = (ao, bo)
        return self._off_cache[key]

    def pack(self, weights: dict, rank: int) -> torch.Tensor:
        """Host-side packing of an adapter dict (``layers.{l}.{t}.A/B``) into a blob (CPU bf16)."""
        layout, n = self.blob_layout(rank)
        blob = torch.empty(n, dtype=torch.bfloat16)
        for l, t, ao, bo, di, do in layout:
            blob[ao:ao + rank * di] = torch.as_tensor(weights[f"layers.{l}.{t}.A"]).reshape(-1).to(torch.bfloat16)
            blob[bo:bo + do * rank] = torch.as_tensor(weights[f"layers.{l}.{t}.B"]).reshape(-1).to(torch.bfloat16)
        return blob

    def install(self, slot: int, blob: torch.Tensor, lora: LoraConfig) -> None:
        """Adopt a device blob (already filled, e.g. by the pre-loader) as slot ``slot``."""
        if lora.rank > self.max_rank or lora.rank % 8:
            raise ValueError(f"rank {lora.rank} must be a multiple of 8 and <= {self.max_rank}")
        if set(lora.targets) - set(self.targets):
            raise ValueError(f"adapter targets {lora.targets} not in pool targets {self.targets}")
        layout, n = self.blob_layout(lora.rank)
        if blob.numel() != n or blob.device != self.device or blob.dtype != torch.bfloat16:
            raise ValueError("blob shape/device/dtype mismatch")
        base = blob.data_ptr()
        a = torch.zeros_like(self.a_ptr[:, :, slot], device="cpu")
        b = torch.zeros_like(a)
        for l, t, ao, bo, _, _ in layout:
            ti = self.targets.index(t)
            if t in lora.targets:
                a[l, ti] = base + 2 * ao
                b[l, ti] = base + 2 * bo
        self.a_ptr[:, :, slot] = a.to(self.device)
        self.b_ptr[:, :, slot] = b.to(self.device)
        self.rank[slot] = lora.rank
        self.scale[slot] = lora.scale
        self.blobs[slot] = blob
        self.configs[slot] = lora
        if self.on_install is not None:
            self.on_install(slot, blob, lora)

    def load(self, slot: int, weights: dict, lora: LoraConfig) -> None:
        blob = self.pack(weights, lora.rank)
        if lora.targets != self.targets:  # untargeted projections: zero A/B, pointer left null
            pass
        self.install(slot, blob.to(self.device), lora)

    def load_random(self, slot: int, lora: LoraConfig, seed: int, std: float = 0.02) -> None:
        """On-device random adapter (A ~ N(0, 1/d_in), B ~ N(0, std)) for large shapes."""
        layout, n = self.blob_layout(lora.rank)
        g = torch.Generator(device=self.device).manual_seed(seed)
        blob = torch.empty(n, dtype=torch.bfloat16, device=self.device)
        for _, _, ao, bo, di, do in layout:
            blob[ao:ao + lora.rank * di] = (torch.randn(lora.rank * di, generator=g, device=self.device)
                                            / math.sqrt(di)).to(torch.bfloat16)
            blob[bo:bo + do * lora.rank] = (torch.randn(do * lora.rank, generator=g, device=self.device)
                                            * std).to(torch.bfloat16)
        self.install(slot, blob, lora)

    def evict(self, slot: int) -> None:
        if self.on_evict is not None:
            self.on_evict(slot)
        self.a_ptr[:, :, slot] = 0
        self.b_ptr[:, :, slot] = 0
        self.rank[slot] = 0
        self.scale[slot] = 0.0
        self.blobs[slot] = None
        self.configs[slot] = None

    def resident_bytes(self) -> int:
        return sum(b.numel() * 2 for b in self.blobs if b is not None)


class MultiLoraModel:
    """Llama backbone + adapter pool + KV pool on one GPU."""

    def __init__(self, cfg: BackboneConfig, *, dtype=torch.bfloat16, device="cuda",
                 max_seqs: int = 64, max_ctx: int = 512, lora_targets=ATTN_TARGETS,
                 n_slots: int = 32, max_rank: int = 16, max_tokens: int = 4096,
                 decode_lora: str = "auto"):
        """``decode_lora`` (bf16): how the decode step's LoRA shrink reads the adapters —
        "stacked": every slot's A rows are appended to the packed q/k/v and o weights, so the
        projection GEMM computes the shrink of every slot in its pass over x (cheapest for small
        pools: no extra launch, but the streamed bytes grow with n_slots * max_rank);
        "gather": a separate shrink kernel reads only the adapters present in the batch
        (slx_lora_shrink; bytes = the distinct adapters', independent of the pool size);
        "auto": stacked while the stacked rows add <= 24 MB per layer (7B, 32 x r16: 16.8 MB),
        gather beyond (e.g. 13B, 128 slots x r64: 335 MB)."""
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("dtype must be bf16 (throughput) or fp32 (parity)")
        self.cfg, self.dtype = cfg, dtype
        self.device = resolve_device(device)
        self.max_seqs, self.max_ctx, self.max_tokens = max_seqs, max_ctx, max_tokens
        self.targets = tuple(lora_targets)
        self.ffn_pad = _round_up(cfg.ffn, 128)
        self.pool = AdapterPool(cfg, self.targets, n_slots, max_rank, self.device)
        nt = len(self.targets)
        self.lora_ws = torch.zeros(max(ops.lora_workspace_bytes(max_tokens, n_slots, max_rank,
                                                                min(nt, 4)), 256) + 256,
                                   dtype=torch.uint8, device=self.device)
        cos, sin = rope_tables(max_ctx, cfg.head_dim, cfg.rope_theta)
        self.cos = torch.from_numpy(cos).to(self.device)
        self.sin = torch.from_numpy(sin).to(self.device)
        kv_shape = (max_seqs, cfg.kv_heads, max_ctx, cfg.head_dim)
        self.k_cache = [torch.zeros(kv_shape, dtype=dtype, device=self.device) for _ in range(cfg.layers)]
        self.v_cache = [torch.zeros(kv_shape, dtype=dtype, device=self.device) for _ in range(cfg.layers)]
        self.seq_len = [0] * max_seqs
        self.free_seqs = list(range(max_seqs))[::-1]
        self.w: dict[str, torch.Tensor] = {}
        # decode shrink inside the projection GEMMs (bf16): stacked A rows of every slot are
        # appended to the packed q/k/v and o weights; the GEMM writes v_all in fp32 as a side
        # output and slx_lora_expand finishes the LoRA term.  Per group: targets, row layout.
        if decode_lora not in ("auto", "stacked", "gather"):
            raise ValueError("decode_lora must be auto, stacked or gather")
        qkv_t = tuple(t for t in ("q", "k", "v") if t in self.targets)
        stacked_bytes = ((len(qkv_t) + ("o" in self.targets)) * n_slots * max_rank *
                         max(cfg.hidden, cfg.q_dim) * 2)
        if decode_lora == "auto":
            decode_lora = "stacked" if stacked_bytes <= (24 << 20) else "gather"
        self.decode_lora = decode_lora if dtype == torch.bfloat16 and self.targets else None
        self.stack = {}
        if self.decode_lora == "stacked":
            if qkv_t:
                self.stack["w_qkv"] = qkv_t
            if "o" in self.targets:
                self.stack["wo"] = ("o",)
        self.use_stacked_decode = bool(self.stack)
        # decode: q/k/v expand fused into the attention kernel, o expand into the post-norm
        self.fuse_expand = True
        # decode: o / down projections as split-K pieces reduced by the following RMSNorm;
        # pieces per tile: o 6 (96 CTAs), down 8 (128 CTAs) — measured best on the 7B step
        # (o at 8: +50 us/step)
        self.splitk_consumer = True
        self.splitk_splits_o, self.splitk_splits_dn = 6, 8
        self._n_sm = None
        # decode: each kernel prefetches the next kernel's first bytes into L2 (MB; 0 = off)
        self.l2_prefetch_mb = 16.0
        self._pf_cache: dict = {}
        self.use_tc_sgmv = dtype == torch.bfloat16   # prefill LoRA as grouped tcgen05 GEMMs
        # prefill: the LoRA expand folded into the backbone GEMM as one extra K block
        self.lora_fold = True
        self._plan_cache: dict = {}   # prefill plans by segment layout (_prefill_plans)
        # prefill batches the fold rejects, up to this many tokens: gathered LoRA kernels
        self.prefill_gather_max_tokens = 1024
        self.prefill_small_lora = "stacked"   # or "gather" (no stacked pool: always gather)
        self.pool.on_install = self._stack_install
        self.pool.on_evict = self._stack_evict

    # ------------------------------------------------------------------ weights
    def load_backbone(self, weights: dict) -> None:
        """Pack a backbone dict (oracle naming, fp32 or bf16) into the device layout."""
        cfg, dev = self.cfg, self.device
        w = {}
        w["embed"] = _to_dev(weights["embed"], dev)
        w["final_norm"] = _to_dev(weights["final_norm"], dev)
        w["lm_head"] = _to_dev(weights["lm_head"], dev)
        for l in range(cfg.layers):
            p = f"layers.{l}."
            g = lambda k: torch.as_tensor(weights[p + k])  # noqa: E731
            w[p + "input_norm"] = _to_dev(g("input_norm"), dev)
            w[p + "post_norm"] = _to_dev(g("post_norm"), dev)
            w[p + "w_qkv"] = _to_dev(torch.cat([g("wq"), g("wk"), g("wv")], 0), dev)
            w[p + "wo"] = _to_dev(g("wo"), dev)
            w[p + "w_gu"] = self._block_gate_up(g("w_gate"), g("w_up")).to(dev)
            down = torch.zeros((cfg.hidden, self.ffn_pad), dtype=torch.bfloat16)
            down[:, :cfg.ffn] = g("w_down").to(torch.bfloat16)
            w[p + "w_down"] = down.to(dev)
        self.w = w
        self._pack()
        self._restack()

    def _block_gate_up(self, gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
        """[gate rows 128 | up rows 128] blocks, zero-padded to ffn_pad (SLX_EPI_SILU_MUL)."""
        f, d = gate.shape
        fp = self.ffn_pad
        gp = torch.zeros((fp, d), dtype=torch.bfloat16, device=gate.device)
        upp = torch.zeros((fp, d), dtype=torch.bfloat16, device=gate.device)
        gp[:f] = gate.to(torch.bfloat16)
        upp[:f] = up.to(torch.bfloat16)
        return torch.stack([gp.view(fp // 128, 128, d), upp.view(fp // 128, 128, d)], 1).reshape(2 * fp, d).contiguous()

    def random_backbone(self, seed: int = 0, std: float = 0.02) -> None:
        """Random-init bf16 backbone generated directly on the device (7B/13B shapes)."""
        cfg, dev = self.cfg, self.device
        g = torch.Generator(device=dev).manual_seed(seed)

        def rn(*shape, s=std, mean=0.0):
            return (torch.randn(*shape, generator=g, device=dev) * s + mean).to(torch.bfloat16)

        w = {"embed": rn(cfg.vocab, cfg.hidden, s=1.0), "final_norm": rn(cfg.hidden, s=0.1, mean=1.0),
             "lm_head": rn(cfg.vocab, cfg.hidden)}
        for l in range(cfg.layers):
            p = f"layers.{l}."
            w[p + "input_norm"] = rn(cfg.hidden, s=0.1, mean=1.0)
            w[p + "post_norm"] = rn(cfg.hidden, s=0.1, mean=1.0)
            w[p + "w_qkv"] = rn(cfg.q_dim + 2 * cfg.kv_dim, cfg.hidden)
            w[p + "wo"] = rn(cfg.hidden, cfg.q_dim)
            w[p + "w_gu"] = self._block_gate_up(rn(cfg.ffn, cfg.hidden), rn(cfg.ffn, cfg.hidden))
            down = torch.zeros((cfg.hidden, self.ffn_pad), dtype=torch.bfloat16, device=dev)
            down[:, :cfg.ffn] = rn(cfg.hidden, cfg.ffn)
            w[p + "w_down"] = down
            if self.dtype == torch.bfloat16:   # pack layer by layer to bound peak memory
                for k in self.PROJ:
                    w[p + k] = ops.pack_weight(w[p + k], self._extra_rows(k))
        if self.dtype == torch.bfloat16:
            w["lm_head"] = ops.pack_weight(w["lm_head"])
        self.w = w
        self._restack()

    PROJ = ("w_qkv", "wo", "w_gu", "w_down")

    def _pack(self) -> None:
        """bf16 mode: re-lay every projection (and lm_head) in the tiled TMA layout."""
        if self.dtype != torch.bfloat16:
            return
        for k in list(self.w):
            if k == "lm_head" or k.split(".")[-1] in self.PROJ:
                self.w[k] = ops.pack_weight(self.w[k], self._extra_rows(k.split(".")[-1]))
        torch.cuda.synchronize(self.device)

    def _extra_rows(self, proj: str) -> int:
        targets = self.stack.get(proj, ())
        return len(targets) * self.pool.n_slots * self.pool.max_rank

    def _stack_rows(self, proj: str, t: str, slot: int) -> int:
        return (self.stack[proj].index(t) * self.pool.n_slots + slot) * self.pool.max_rank

    def _stack_install(self, slot: int, blob: torch.Tensor, lora) -> None:
        if not self.stack or not self.w:
            return
        layout, _ = self.pool.blob_layout(lora.rank)
        R = self.pool.max_rank
        for l, t, ao, _bo, di, _do in layout:
            for proj, ts in self.stack.items():
                if t not in ts:
                    continue
                pw = self.w[f"layers.{l}.{proj}"]
                row0 = pw.n + self._stack_rows(proj, t, slot)
                if t in lora.targets:
                    a = blob[ao:ao + lora.rank * di].view(lora.rank, di)
                    ops.pack_rows(pw, a, lora.rank, row0)
                    if lora.rank < R:
                        ops.pack_rows(pw, None, R - lora.rank, row0 + lora.rank)
                else:
                    ops.pack_rows(pw, None, R, row0)

    def _restack(self) -> None:
        """(Re)write the stacked A rows of every resident adapter (backbone loaded later)."""
        for slot, blob in enumerate(self.pool.blobs):
            if blob is not None:
                self._stack_install(slot, blob, self.pool.configs[slot])

    def _stack_evict(self, slot: int) -> None:
        if not self.stack or not self.w:
            return
        for l in range(self.cfg.layers):
            for proj, ts in self.stack.items():
                pw = self.w[f"layers.{l}.{proj}"]
                for t in ts:
                    ops.pack_rows(pw, None, self.pool.max_rank, pw.n + self._stack_rows(proj, t, slot))

    def memory_ledger(self) -> dict:
        """Device bytes this model holds, in the categories the reference's ResidencyLedger
        books per GPU (``/root/reference/pkg/src/slorasim/ledger.py:47-182``): the one backbone
        copy (``ledger.py:130-134``), the adapter residents (pool slots plus their stacked
        decode-shrink rows inside the packed q/k/v/o weights), the KV pool (one fixed
        ``kv_slot_bytes`` reservation per sequence slot) and workspaces.  ``total`` equals the
        growth of the caching allocator's requested bytes from constructing and loading the
        model (tests/test_gpu_runtime.py)."""
        lib = _lib.load()
        seen: set = set()
        cats = {"backbone": 0, "adapter_pool": 0, "adapter_stacked_rows": 0, "kv_pool": 0,
                "workspace": 0}
        n_storages = [0]

        def add(cat, t, stacked: int = 0):
            t = getattr(t, "data", t)
            if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
                return
            st = t.untyped_storage()
            if st.data_ptr() in seen:
                return
            seen.add(st.data_ptr())
            nb = st.nbytes()
            cats[cat] += nb - stacked
            cats["adapter_stacked_rows"] += stacked
            n_storages[0] += 1

        for t in self.w.values():
            stacked = 0
            if isinstance(t, ops.PackedWeight) and t.n_extra:
                stacked = t.data.numel() * 2 - int(lib.slx_packed_weight_elems(t.n, t.k)) * 2
            add("backbone", t, stacked)
        for b in self.pool.blobs:
            if b is not None:
                add("adapter_pool", b)
        for t in self.k_cache + self.v_cache:
            add("kv_pool", t)

        def walk(obj, depth=0):
            if depth > 2:
                return
            for v in (obj.values() if isinstance(obj, dict) else
                      obj if isinstance(obj, (list, tuple)) else vars(obj).values()):
                if isinstance(v, torch.Tensor) or isinstance(v, ops.PackedWeight):
                    add("workspace", v)
                elif isinstance(v, (dict, list, tuple)):
                    walk(v, depth + 1)
        walk(self)
        walk(self.pool)
        kv_slot = self.cfg.kv_bytes_per_token() * self.max_ctx * (2 if self.dtype == torch.float32 else 1)
        return {**cats, "total": sum(cats.values()), "storages": n_storages[0],
                "kv_slot_bytes": kv_slot, "max_seqs": self.max_seqs}

    def backbone_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.w.values())

    # ------------------------------------------------------------------ sequences
    def alloc_seq(self) -> int:
        if not self.free_seqs:
            raise RuntimeError("KV pool exhausted")
        s = self.free_seqs.pop()
        self.seq_len[s] = 0
        return s

    def free_seq(self, s: int) -> None:
        self.seq_len[s] = 0
        self.free_seqs.append(s)

    # ------------------------------------------------------------------ forward
    def _gemm(self, a, w, out=None, residual=None, silu=False, out_dtype=None, prefetch=None):
        if self.dtype == torch.bfloat16:
            epi = EPI_SILU_MUL if silu else (EPI_RESIDUAL if residual is not None else 0)
            return ops.gemm(a, w, out, epilogue=epi, residual=residual, out_dtype=out_dtype,
                            prefetch=prefetch)
        assert not silu
        return ops.gemm_f32(a, w, out, residual=residual)

    def _lora(self, y, x, layer: int, names, cols, d_in=None):
        """Apply LoRA of targets ``names`` with output column maps ``cols``."""
        idx = [i for i, t in enumerate(self.targets) if t in names]
        if not idx:
            return
        specs = []
        for i in idx:
            t = self.targets[i]
            off, blk, stride = cols[t]
            specs.append((self.pool.a_ptr[layer, i], self.pool.b_ptr[layer, i],
                          self.cfg.target_dims(t)[1], off, blk, stride))
        ops.lora_apply(y, x, d_in if d_in is not None else x.shape[1], self.pool.rank,
                       self.pool.scale, self.pool.max_rank, ops.make_targets(specs), self.lora_ws)

    def _sgmv_plan(self, segments, slot_host):
        """Grouped-GEMM tile tables for the prefill LoRA (SGMV on tcgen05), built once per
        forward: per launch (<= 16 adapter groups) the shrink tiles and, per distinct d_out,
        the expand tiles, uploaded to the device in one copy each."""
        by_slot: dict = {}
        for tok0, n, _seq, _p0 in segments:
            a = int(slot_host[tok0])
            if a >= 0 and self.pool.configs[a] is not None:
                by_slot.setdefault(a, []).append((tok0, n))
        slots = sorted(by_slot)
        douts = sorted({self.cfg.target_dims(t)[1] for t in self.targets})
        launches = []
        for c in range(0, len(slots), ops.GROUP_MAX):
            chunk = slots[c:c + ops.GROUP_MAX]
            shrink, expand = [], {do: [] for do in douts}
            for gi, a in enumerate(chunk):
                for tok0, n in by_slot[a]:
                    for m0 in range(tok0, tok0 + n, 128):
                        mr = min(128, tok0 + n - m0)
                        shrink.append((gi, m0, mr, 0))
                        for do in douts:
                            expand[do] += [(gi, m0, mr, n0) for n0 in range(0, do, 256)]
            dev = lambda rows: torch.tensor(rows, dtype=torch.int32).reshape(-1, 4).to(self.device)  # noqa: E731
            launches.append((chunk, dev(shrink), {do: dev(v) for do, v in expand.items()}))
        return launches

    def _fold_plan(self, segments, slot_host, T: int):
        """Prefill LoRA folded into the backbone GEMMs: grouped tiles of the qkv / o GEMMs
        (segment-aligned 128-row blocks, group = the adapter's index, -1 = none) and the shrink
        tiles.  None when the batch does not fit the fold (> 16 adapters, partial target sets,
        short segments that would waste tensor-core rows)."""
        cfg = self.cfg
        if set(self.targets) != {"q", "k", "v", "o"} or self.pool.max_rank > 64:
            return None
        if cfg.q_dim % 256 or cfg.kv_dim % 256 or cfg.hidden % 256:
            return None
        slots = sorted({int(slot_host[t0]) for t0, _n, _s, _p in segments
                        if int(slot_host[t0]) >= 0 and self.pool.configs[int(slot_host[t0])] is not None})
        if len(slots) > ops.GROUP_MAX or any(set(self.pool.configs[a].targets) != set(self.targets)
                                             for a in slots):
            return None
        gi = {a: i for i, a in enumerate(slots)}
        nq = cfg.q_dim + 2 * cfg.kv_dim
        mblocks, sh = [], []
        for tok0, n, _seq, _p0 in segments:
            g = gi.get(int(slot_host[tok0]), -1)
            for m0 in range(tok0, tok0 + n, 128):
                mblocks.append((g, m0, min(128, tok0 + n - m0)))
                if g >= 0:
                    sh.append((g, m0, min(128, tok0 + n - m0), 0))
        if len(mblocks) > 1.25 * ((T + 127) // 128) + 1:
            return None
        # rasterised tile order (groups of 16 row blocks x every column tile): the co-resident
        # CTAs share a few activation row blocks and weight tiles in L2
        def raster(n_cols):
            out = []
            for r0 in range(0, len(mblocks), 16):
                grp = mblocks[r0:r0 + 16]
                for n0 in range(0, n_cols, 256):
                    out += [(g, m0, mr, n0) for g, m0, mr in grp]
            return out
        tq, to = raster(nq), raster(cfg.hidden)
        dev = lambda rows: torch.tensor(rows, dtype=torch.int32).reshape(-1, 4).to(self.device)  # noqa: E731
        return slots, dev(tq), dev(to), dev(sh) if sh else None

    def _fold_lora(self, layer: int, slots, proj: str):
        """(A groups for the shrink per target, B pointers adapter-major, ranks)."""
        names = ("q", "k", "v") if proj == "w_qkv" else ("o",)
        ga = {t: [] for t in names}
        bp, ranks = [], []
        for a in slots:
            lo = self.pool.configs[a]
            base = self.pool.blobs[a].data_ptr()
            ranks.append(lo.rank)
            for t in names:
                di, do = self.cfg.target_dims(t)
                ao, bo = self.pool.offsets(lo.rank, layer, t)
                ga[t].append((base + 2 * ao, lo.rank, di, di, lo.scale))
                bp.append(base + 2 * bo)
        return ga, bp, ranks

    def _sgmv_tc(self, y, x, layer: int, names, cols, plan, v_buf) -> bool:
        """Prefill LoRA for contiguous targets via two grouped tcgen05 GEMMs per target:
        v = scale * x A^T (shrink, bf16 [T, 64]) then y[:, off:] += v B^T (expand)."""
        idx = [i for i, t in enumerate(self.targets) if t in names]
        if not idx:
            return True
        R = 64
        for i in idx:
            t = self.targets[i]
            _off, blk, _stride = cols[t]
            if blk != self.cfg.target_dims(t)[1] or self.pool.max_rank > R:
                return False
        for chunk, sh_tiles, ex_tiles in plan:
            for i in idx:
                t = self.targets[i]
                off, _blk, _stride = cols[t]
                di, do = self.cfg.target_dims(t)
                ga, gb = [], []
                for a in chunk:
                    lo = self.pool.configs[a]
                    ao, bo = self.pool.offsets(lo.rank, layer, t)
                    base = self.pool.blobs[a].data_ptr()
                    ga.append((base + 2 * ao, lo.rank, di, di, lo.scale))
                    gb.append((base + 2 * bo, do, lo.rank, lo.rank, 1.0))
                ops.gemm_grouped(x, di, ga, sh_tiles, v_buf, R)
                yv = y[:, off:off + do]
                ops.gemm_grouped(v_buf, R, gb, ex_tiles[do], yv, do, residual=yv)
        return True

    def _expand(self, y, v_all, layer: int, proj: str, cols) -> None:
        specs, offs = [], []
        for t in self.stack[proj]:
            i = self.targets.index(t)
            off, blk, stride = cols[t]
            specs.append((self.pool.a_ptr[layer, i], self.pool.b_ptr[layer, i],
                          self.cfg.target_dims(t)[1], off, blk, stride))
            offs.append(self._stack_rows(proj, t, 0))
        ops.lora_expand(y, v_all, self.pool.rank, self.pool.scale, self.pool.max_rank,
                        ops.make_targets(specs), offs, self.lora_ws)

    def _pf(self, key, *tensors):
        """Cached slx_l2_prefetch of the first l2_prefetch_mb MB (split over the tensors)."""
        if self.l2_prefetch_mb <= 0:
            return None
        if key not in self._pf_cache:
            n = int(self.l2_prefetch_mb * (1 << 20)) // len(tensors)
            self._pf_cache[key] = ops.l2_prefetch(*[(getattr(t, "data", t), n) for t in tensors])
        return self._pf_cache[key]

    def _pf_all(self, key, t):
        """slx_l2_prefetch of a whole (packed) weight (spread over a long kernel)."""
        if self.l2_prefetch_mb <= 0:
            return None
        if key not in self._pf_cache:
            d = getattr(t, "data", t)
            self._pf_cache[key] = ops.l2_prefetch((d, d.numel() * d.element_size()))
        return self._pf_cache[key]

    def _delta(self, layer: int, proj: str, v_all, slot, cols):
        """slx_lora_delta of the stacked targets of ``proj`` (fused decode expand)."""
        tg = []
        for t in self.stack[proj]:
            i = self.targets.index(t)
            tg.append((self.pool.b_ptr[layer, i], self._stack_rows(proj, t, 0), cols[t][0],
                       self.cfg.target_dims(t)[1]))
        return ops.make_delta(v_all, slot, self.pool.rank, self.pool.scale, self.pool.max_rank, tg)

    def _gather_targets(self, layer: int, names):
        """(targets array, v column offsets) of the gathered shrink / delta of ``names``."""
        idx = [i for i, t in enumerate(self.targets) if t in names]
        specs = [(self.pool.a_ptr[layer, i], self.pool.b_ptr[layer, i],
                  self.cfg.target_dims(self.targets[i])[1], 0, 1, 1) for i in idx]
        return idx, ops.make_targets(specs), [k * self.pool.max_rank for k in range(len(idx))]

    def _gather_shrink(self, layer: int, names, x, v) -> None:
        """Gathered decode shrink of targets ``names`` on input x into v (compact:
        [T, len(names) * max_rank], only the batch's adapters read)."""
        idx, targets, offs = self._gather_targets(layer, names)
        if idx:
            ops.lora_shrink(v, x, self.pool.rank, self.pool.max_rank, targets, offs, self.lora_ws)

    def _gather_expand(self, layer: int, names, y, v, cols) -> None:
        """y[t, col] += scale * v . B^T for the gathered v of targets ``names`` (in place; the
        expand kernel reads each present adapter's B rows once per plan tile)."""
        idx = [i for i, t in enumerate(self.targets) if t in names]
        if not idx:
            return
        specs = [(self.pool.a_ptr[layer, i], self.pool.b_ptr[layer, i],
                  self.cfg.target_dims(self.targets[i])[1], *cols[self.targets[i]]) for i in idx]
        ops.lora_expand(y, v, self.pool.rank, self.pool.scale, self.pool.max_rank,
                        ops.make_targets(specs), [k * self.pool.max_rank for k in range(len(idx))],
                        self.lora_ws, v_slot_stride=0)

    @staticmethod
    def segments_of(pos, seq) -> list:
        """Host (tok0, n, seq, pos0) runs of consecutive positions of one sequence."""
        pos, seq = np.asarray(pos, dtype=np.int64), np.asarray(seq, dtype=np.int64)
        if pos.size == 0:
            return []
        # a run breaks where the sequence changes or the position does not advance by one
        brk = np.flatnonzero((seq[1:] != seq[:-1]) | (pos[1:] != pos[:-1] + 1)) + 1
        starts = np.concatenate([[0], brk])
        lens = np.diff(np.concatenate([starts, [pos.size]]))
        return [(int(a), int(n), int(q), int(p0))
                for a, n, q, p0 in zip(starts, lens, seq[starts], pos[starts])]

    def _sk_splits(self, n_out: int, k: int, pieces: int) -> int:
        """Split-K pieces of a decode projection (o, down): the tuned count (7B: o 6, down 8)
        unless its grid -- ceil(n_out / 256) tiles x pieces, one tcgen05 CTA per SM -- exceeds
        the SMs; then pieces filling ~70 % of them, since a second wave doubles the launch
        (13B down: 20 x 8 = 160 CTAs -> 20 x 5; pool decode 10.06 -> 9.45 ms/step,
        exp/sk_splits_13b.py)."""
        tiles = (n_out + 255) // 256
        s = max(1, min(pieces, k // 64))
        if self._n_sm is None:
            self._n_sm = ops.sm_count()
        if tiles * s > self._n_sm:
            s = max(1, int(0.7 * self._n_sm) // tiles)
        return s

    def _decode_fast(self, T: int) -> bool:
        """The bf16 decode step of fused kernels (split-K consumers, fused LoRA expands)."""
        d = self.cfg.hidden
        return (self.dtype == torch.bfloat16 and self.splitk_consumer and self.fuse_expand
                and T <= 128 and d % 256 == 0 and d <= 5120
                and set(self.targets) <= {"q", "k", "v", "o"}
                and (not self.targets or (self.decode_lora == "gather") or
                     (self.use_stacked_decode and self.pool.max_rank <= 16)))

    def forward(self, tokens, pos, seq, slot, logit_rows=None, decode: bool = False,
                segments=None, slot_host=None) -> torch.Tensor:
        """Token-major mixed batch.  tokens/pos/seq/slot: device int32 [T].
        ``decode``: every token is the next position of its own sequence, so RoPE, the KV
        append and attention run as one fused kernel per layer.  The caller guarantees
        pos < max_ctx (MultiLoraModel.prefill/decode and the serving runtime check it).
        ``slot_host``: the same per-token slots on the host when the caller has them (prefill
        plans need them; otherwise they are read back from the device, a stream sync).
        Returns logits (fp32) for ``logit_rows`` (device int64) or for every token."""
        T = tokens.numel()
        if T > self.max_tokens:
            raise ValueError(f"batch of {T} tokens exceeds max_tokens={self.max_tokens}")
        if decode and self._decode_fast(T):
            return self._forward_decode(tokens, pos, seq, slot, logit_rows)
        return self._forward_general(tokens, pos, seq, slot, logit_rows, decode, segments,
                                     slot_host)

    def _forward_decode(self, tokens, pos, seq, slot, logit_rows):
        """bf16 decode step: per layer [RMSNorm(+ pieces of the previous down projection)] ->
        [gathered shrink] -> q/k/v GEMM (stacked shrink rows as an fp32 side output) ->
        RoPE + KV append + attention with the q/k/v LoRA expand fused -> [gathered shrink] ->
        o GEMM as split-K pieces -> RMSNorm consuming the pieces + the o LoRA expand ->
        gate/up GEMM with SiLU*mul -> down GEMM as split-K pieces (consumed by the next norm)."""
        cfg, w, dt, dev = self.cfg, self.w, self.dtype, self.device
        T = tokens.numel()
        d, qd, kvd = cfg.hidden, cfg.q_dim, cfg.kv_dim
        R = self.pool.max_rank
        x = torch.empty((T, d), dtype=dt, device=dev)
        h = torch.empty((T, d), dtype=dt, device=dev)
        qkv = torch.empty((T, qd + 2 * kvd), dtype=dt, device=dev)
        attn = torch.empty((T, qd), dtype=dt, device=dev)
        mlp = torch.empty((T, self.ffn_pad), dtype=dt, device=dev)
        stacked = self.decode_lora == "stacked" and bool(self.stack)
        gather = self.decode_lora == "gather"
        qkv_names = tuple(t for t in ("q", "k", "v") if t in self.targets)
        v_qkv = (torch.empty((T, self._extra_rows("w_qkv")), dtype=torch.float32, device=dev)
                 if stacked and "w_qkv" in self.stack else None)
        if gather:
            v_g = torch.empty((T, max(1, len(qkv_names)) * R), dtype=torch.float32, device=dev)
            v_go = torch.empty((T, R), dtype=torch.float32, device=dev)
        S = self._sk_splits(d + self._extra_rows("wo"), cfg.q_dim, self.splitk_splits_o)
        S_dn = self._sk_splits(d, self.ffn_pad, self.splitk_splits_dn)
        part_o = torch.empty(ops.splitk_bytes(T, d + self._extra_rows("wo"), S) // 4,
                             dtype=torch.float32, device=dev)
        part_dn = torch.empty(ops.splitk_bytes(T, d, S_dn) // 4, dtype=torch.float32, device=dev)
        qkv_cols = {"q": (0, qd, qd), "k": (qd, kvd, kvd), "v": (qd + kvd, kvd, kvd)}
        ops.embedding(x, w["embed"], tokens)
        if self.targets:
            ops.lora_plan_tokens(slot, self.pool.n_slots, self.lora_ws)
        pending = None   # split-K pieces of the down projection, consumed by the next norm
        for l in range(cfg.layers):
            p = f"layers.{l}."
            if pending is None:
                ops.rmsnorm(h, x, w[p + "input_norm"], cfg.rms_eps)
            else:
                ops.rmsnorm_fused(h, x, w[p + "input_norm"], cfg.rms_eps, pending)
            # L2 prefetch chain: every kernel requests the first bytes of its successor
            nxt = f"layers.{l + 1}.w_qkv" if l + 1 < cfg.layers else "lm_head"
            pf_qkv = self._pf(("kv", l), self.k_cache[l], self.v_cache[l])
            pf_att = self._pf(p + "wo", w[p + "wo"])
            pf_gu = self._pf(p + "w_down", w[p + "w_down"])
            pf_o = self._pf(p + "w_gu", w[p + "w_gu"])
            pf_dn = self._pf(nxt, w[nxt])
            # q / k / v
            d_qkv = None
            if stacked and "w_qkv" in self.stack:
                ops.gemm(h, w[p + "w_qkv"], qkv, side=v_qkv, prefetch=pf_qkv)
                d_qkv = self._delta(l, "w_qkv", v_qkv, slot, qkv_cols)
            else:
                if gather and qkv_names:
                    self._gather_shrink(l, qkv_names, h, v_g)
                ops.gemm(h, w[p + "w_qkv"], qkv, prefetch=pf_qkv)
                if gather and qkv_names:   # q/k/v deltas added in place (== the fused expand)
                    self._gather_expand(l, qkv_names, qkv, v_g, qkv_cols)
            ops.rope_attention_decode(attn, qkv, cfg.heads, cfg.kv_heads, cfg.head_dim, pos, seq,
                                      self.cos, self.sin, self.k_cache[l], self.v_cache[l],
                                      lora=d_qkv, prefetch=pf_att)
            # o (split-K pieces) -> residual + o LoRA + post-attention RMSNorm
            d_o = None
            if gather and "o" in self.targets:
                self._gather_shrink(l, ("o",), attn, v_go)
            sk_o = ops.gemm_splitk(attn, w[p + "wo"], S, part_o, prefetch=pf_o)
            if gather and "o" in self.targets:   # the o delta into the residual before the norm
                self._gather_expand(l, ("o",), x, v_go, {"o": (0, d, d)})
            if stacked and "wo" in self.stack:
                d_o = self._delta(l, "wo", None, slot, {"o": (0, d, d)})
            ops.rmsnorm_fused(h, x, w[p + "post_norm"], cfg.rms_eps, sk_o, d_o)
            # MLP
            ops.gemm(h, w[p + "w_gu"], mlp, epilogue=EPI_SILU_MUL, prefetch=pf_gu)
            pending = ops.gemm_splitk(mlp, w[p + "w_down"], S_dn, part_dn, prefetch=pf_dn)
        hn = torch.empty_like(x)
        ops.rmsnorm_fused(hn, x, w["final_norm"], cfg.rms_eps, pending)
        if logit_rows is not None:
            hn = hn.index_select(0, logit_rows)
        return ops.gemm(hn, w["lm_head"], out_dtype=torch.float32)

    def _small_prefill(self, T: int) -> bool:
        """Prefill LoRA through the gathered / stacked decode kernels (batches the fold
        declines, up to prefill_gather_max_tokens tokens)."""
        return (T <= self.prefill_gather_max_tokens and set(self.targets) <= {"q", "k", "v", "o"}
                and self.pool.max_rank <= 64)

    def _prefill_plans(self, segments, slot_host, T: int, flash: bool, sgmv: bool):
        """(flash plan, LoRA-fold plan, SGMV plan) of a segmented prefill batch, cached by the
        segment layout and the segments' adapter slots (a serving loop re-plans only when the
        batch shape changes; the plans are device tensors built once)."""
        slots = tuple(int(slot_host[sg[0]]) for sg in segments) if sgmv else None
        key = (tuple(tuple(int(v) for v in sg) for sg in segments), slots, T, flash, sgmv,
               self.lora_fold)
        hit = self._plan_cache.get(key)
        if hit is not None:
            return hit
        plan = ops.prefill_plan(segments, self.cfg.heads, self.device) if flash else None
        fold = sgmv_plan = None
        if sgmv:
            if self.lora_fold:
                fold = self._fold_plan(segments, slot_host, T)
            if fold is None and not self._small_prefill(T):   # the small path plans on device
                sgmv_plan = self._sgmv_plan(segments, slot_host)
        if len(self._plan_cache) >= 16:
            self._plan_cache.pop(next(iter(self._plan_cache)))
        self._plan_cache[key] = (plan, fold, sgmv_plan)
        return plan, fold, sgmv_plan

    def _forward_general(self, tokens, pos, seq, slot, logit_rows, decode, segments, slot_host=None):
        """Prefill (bf16: tcgen05 GEMMs with the LoRA folded / grouped SGMV, flash attention)
        and the fp32 parity mode (decode included)."""
        cfg, w, dt = self.cfg, self.w, self.dtype
        T = tokens.numel()
        dev = self.device
        d, qd, kvd = cfg.hidden, cfg.q_dim, cfg.kv_dim
        x = torch.empty((T, d), dtype=dt, device=dev)
        h = torch.empty((T, d), dtype=dt, device=dev)
        qkv = torch.empty((T, qd + 2 * kvd), dtype=dt, device=dev)
        attn = torch.empty((T, qd), dtype=dt, device=dev)
        mlp = torch.empty((T, self.ffn_pad), dtype=dt, device=dev)
        fused_silu = dt == torch.bfloat16 and not ({"gate", "up"} & set(self.targets))
        gu = None if fused_silu else torch.empty((T, 2 * self.ffn_pad), dtype=dt, device=dev)
        # small bf16 batches with a stacked pool: shrink as the GEMM side output + expand kernel
        stacked = self.use_stacked_decode and T <= 128 and bool(self.stack)
        if stacked:
            v_qkv = (torch.empty((T, self._extra_rows("w_qkv")), dtype=torch.float32, device=dev)
                     if "w_qkv" in self.stack else None)
            v_o = (torch.empty((T, self._extra_rows("wo")), dtype=torch.float32, device=dev)
                   if "wo" in self.stack else None)
        flash = (segments is not None and not decode and dt == torch.bfloat16
                 and cfg.head_dim == 128)
        sgmv = (segments is not None and not decode and dt == torch.bfloat16 and bool(self.targets)
                and self.use_tc_sgmv and not stacked)
        plan = fold = sgmv_plan = None
        if flash or sgmv:
            if sgmv and slot_host is None:
                slot_host = slot.cpu().numpy()
            plan, fold, sgmv_plan = self._prefill_plans(segments, slot_host, T, flash, sgmv)
        # RoPE + KV append fused into the q/k/v GEMM's epilogue (LoRA-fold path, head_dim 128)
        rope_fused = (fold is not None and not decode and cfg.head_dim == 128
                      and (cfg.heads * 128) % 256 == 0 and (cfg.kv_heads * 128) % 256 == 0)
        # short-segment batches the fold rejects (a serving round's merged small prompts): the
        # gathered shrink / expand kernels of the decode path, parallel over token tiles, instead
        # of per-segment grouped GEMMs whose few CTAs each walk the whole K
        small = sgmv and fold is None and self._small_prefill(T)
        if small and self.prefill_small_lora == "stacked" and self.use_stacked_decode and self.stack:
            # or the stacked shrink as the projection GEMM's side output (no shrink launches)
            stacked, small, sgmv_plan = True, False, None
            v_qkv = (torch.empty((T, self._extra_rows("w_qkv")), dtype=torch.float32, device=dev)
                     if "w_qkv" in self.stack else None)
            v_o = (torch.empty((T, self._extra_rows("wo")), dtype=torch.float32, device=dev)
                   if "wo" in self.stack else None)
        gather_pf = small
        if gather_pf:
            qkv_names = tuple(t for t in ("q", "k", "v") if t in self.targets)
            v_g = torch.empty((T, max(1, len(qkv_names)) * self.pool.max_rank), dtype=torch.float32,
                              device=dev)
            sgmv_plan = None
        if sgmv:
            if fold is None:
                v_buf = torch.empty((T, 64), dtype=dt, device=dev)
            else:
                v_qkv_f = torch.zeros((T, 192), dtype=dt, device=dev)
                v_o_f = torch.zeros((T, 64), dtype=dt, device=dev)
                bq = [cfg.q_dim, cfg.kv_dim, cfg.kv_dim]
        ops.embedding(x, w["embed"], tokens)
        if self.targets:
            ops.lora_plan_tokens(slot, self.pool.n_slots, self.lora_ws)
        qkv_cols = {"q": (0, qd, qd), "k": (qd, kvd, kvd), "v": (qd + kvd, kvd, kvd)}
        for l in range(cfg.layers):
            p = f"layers.{l}."
            ops.rmsnorm(h, x, w[p + "input_norm"], cfg.rms_eps)
            if fold is not None:
                ga, bp, rk = self._fold_lora(l, fold[0], "w_qkv")
                if fold[3] is not None:   # q, k, v shrinks in one pass over h
                    segs = [e for a in range(len(fold[0])) for e in (ga["q"][a], ga["k"][a], ga["v"][a])]
                    ops.gemm_grouped(h, cfg.hidden, segs, fold[3], v_qkv_f, 192, n_seg=3)
                ops.gemm_lorafold(h, w[p + "w_qkv"], qkv, fold[1], v_qkv_f,
                                  [0, cfg.q_dim, cfg.q_dim + cfg.kv_dim], bp, bq, rk,
                                  rope=(ops.rope_kv(cfg.heads, cfg.kv_heads, cfg.head_dim, pos, seq,
                                                    self.cos, self.sin, self.k_cache[l],
                                                    self.v_cache[l]) if rope_fused else None))
            elif stacked and "w_qkv" in self.stack:
                ops.gemm(h, w[p + "w_qkv"], qkv, side=v_qkv)
                self._expand(qkv, v_qkv, l, "w_qkv", qkv_cols)
            elif gather_pf:
                self._gemm(h, w[p + "w_qkv"], qkv)
                if qkv_names:
                    self._gather_shrink(l, qkv_names, h, v_g)
                    self._gather_expand(l, qkv_names, qkv, v_g, qkv_cols)
            else:
                self._gemm(h, w[p + "w_qkv"], qkv)
                if not (sgmv_plan is not None and
                        self._sgmv_tc(qkv, h, l, ("q", "k", "v"), qkv_cols, sgmv_plan, v_buf)):
                    self._lora(qkv, h, l, ("q", "k", "v"), qkv_cols)
            if decode:
                ops.rope_attention_decode(attn, qkv, cfg.heads, cfg.kv_heads, cfg.head_dim, pos,
                                          seq, self.cos, self.sin, self.k_cache[l], self.v_cache[l])
            else:
                if not (rope_fused and fold is not None):
                    ops.rope_kv_write(qkv, cfg.heads, cfg.kv_heads, cfg.head_dim, pos, seq, self.cos,
                                      self.sin, self.k_cache[l], self.v_cache[l])
                if flash:
                    ops.attention_prefill(attn, qkv, cfg.heads, cfg.kv_heads, cfg.head_dim, plan,
                                          self.k_cache[l], self.v_cache[l])
                else:
                    ops.attention(attn, qkv, cfg.heads, cfg.kv_heads, cfg.head_dim, pos, seq,
                                  self.k_cache[l], self.v_cache[l])
            if fold is not None:
                ga, bp, rk = self._fold_lora(l, fold[0], "wo")
                if fold[3] is not None:
                    ops.gemm_grouped(attn, cfg.q_dim, ga["o"], fold[3], v_o_f, 64)
                ops.gemm_lorafold(attn, w[p + "wo"], x, fold[2], v_o_f, [0], bp, [cfg.hidden], rk,
                                  residual=x)
            elif stacked and "wo" in self.stack:
                ops.gemm(attn, w[p + "wo"], x, epilogue=EPI_RESIDUAL, residual=x, side=v_o)
                self._expand(x, v_o, l, "wo", {"o": (0, d, d)})
            elif gather_pf:
                self._gemm(attn, w[p + "wo"], x, residual=x)
                if "o" in self.targets:
                    self._gather_shrink(l, ("o",), attn, v_g)
                    self._gather_expand(l, ("o",), x, v_g, {"o": (0, d, d)})
            else:
                self._gemm(attn, w[p + "wo"], x, residual=x)
                if not (sgmv_plan is not None and
                        self._sgmv_tc(x, attn, l, ("o",), {"o": (0, d, d)}, sgmv_plan, v_buf)):
                    self._lora(x, attn, l, ("o",), {"o": (0, d, d)})
            ops.rmsnorm(h, x, w[p + "post_norm"], cfg.rms_eps)
            if fused_silu:
                self._gemm(h, w[p + "w_gu"], mlp, silu=True)
            else:
                self._gemm(h, w[p + "w_gu"], gu)
                self._lora(gu, h, l, ("gate", "up"), {"gate": (0, 128, 256), "up": (128, 128, 256)})
                ops.silu_mul_blocked(mlp, gu, self.ffn_pad)
            self._gemm(mlp, w[p + "w_down"], x, residual=x)
            self._lora(x, mlp, l, ("down",), {"down": (0, d, d)}, d_in=cfg.ffn)
        rows = x if logit_rows is None else x.index_select(0, logit_rows)
        hn = torch.empty_like(rows)
        ops.rmsnorm(hn, rows, w["final_norm"], cfg.rms_eps)
        if dt == torch.bfloat16:
            return self._gemm(hn, w["lm_head"], out_dtype=torch.float32)
        return self._gemm(hn, w["lm_head"])

    # ------------------------------------------------------------------ request-level API
    def prefill(self, prompts, adapter_slots):
        """Start one sequence per prompt (one mixed, adapter-segmented batch).
        Returns (seq_ids, last-token logits [n, V] fp32)."""
        seqs = [self.alloc_seq() for _ in prompts]
        toks, pos, sq, sl, last = [], [], [], [], []
        for s, p, a in zip(seqs, prompts, adapter_slots):
            L = len(p)
            if L + self.seq_len[s] > self.max_ctx:
                raise ValueError("prompt exceeds max_ctx")
            toks += list(p)
            pos += list(range(self.seq_len[s], self.seq_len[s] + L))
            sq += [s] * L
            sl += [a] * L
            last.append(len(toks) - 1)
            self.seq_len[s] += L
        dev = self.device
        i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
        logits = self.forward(i32(toks), i32(pos), i32(sq), i32(sl),
                              torch.tensor(last, dtype=torch.int64, device=dev),
                              segments=self.segments_of(pos, sq), slot_host=np.asarray(sl))
        return seqs, logits

    def decode(self, seqs, tokens, adapter_slots) -> torch.Tensor:
        pos = []
        for s in seqs:
            if self.seq_len[s] >= self.max_ctx:
                raise ValueError("sequence reached max_ctx")
            pos.append(self.seq_len[s])
            self.seq_len[s] += 1
        dev = self.device
        i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
        return self.forward(i32(list(tokens)), i32(pos), i32(list(seqs)), i32(list(adapter_slots)),
                            decode=len(set(seqs)) == len(seqs))

    def argmax(self, logits: torch.Tensor) -> torch.Tensor:
        out = torch.empty(logits.shape[0], dtype=torch.int32, device=logits.device)
        return ops.argmax(out, logits)

    def generate(self, prompts, adapter_slots, n_new: int, return_logits: bool = False):
        """Greedy decode; returns tokens [n, n_new] (np.int64) (+ per-step logits)."""
        seqs, logits = self.prefill(prompts, adapter_slots)
        toks, all_logits = [], []
        try:
            for step in range(n_new):
                if return_logits:
                    all_logits.append(logits.float().cpu())
                nxt = self.argmax(logits)
                toks.append(nxt.cpu().numpy().astype(np.int64))
                if step + 1 < n_new:
                    logits = self.decode(seqs, toks[-1].tolist(), adapter_slots)
        finally:
            for s in seqs:
                self.free_seq(s)
        out = np.stack(toks, 1)
        if return_logits:
            return out, torch.stack(all_logits, 1).numpy()
        return out
