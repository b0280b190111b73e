"""Decode engine: one CUDA-graph-captured mixed-adapter decode step per GPU.

The reference advances every co-running batch by ``decode_ms_per_token * M`` per
token (``/root/reference/pkg/src/slorasim/engine.py:888,909``, processor sharing
``engine.py:259-278``).  Here all sequences resident on a GPU — whatever function
(adapter) they belong to — advance together in ONE step: embedding, the layers of
tcgen05 GEMMs + multi-LoRA + attention, lm_head and argmax, replayed as a single
CUDA graph so the ~230 kernel launches cost one graph launch.

* ``DecodeGraph`` — a static batch of ``B`` rows whose per-step inputs (token, position,
  KV sequence slot, adapter slot) live in ONE device int32 tensor ``inp[4, B]``, so an
  end-to-end step is one pinned H2D copy, one replay and one D2H copy of the sampled tokens.
* ``DecodeBuckets`` — graphs for a ladder of batch sizes (1, 2, 4, ... 64) used by the
  serving runtime: a step of ``n`` active sequences replays the smallest bucket ``>= n`` with
  the spare rows pointed at a reserved padding sequence slot (adapter -1), whose KV rows are
  scratch.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .model import MultiLoraModel


class DecodeGraph:
    """Static-shape decode step for ``len(seqs)`` rows.

    ``fixed_pos``: if given, every replay decodes at this position (the KV append rewrites
    the same row), which keeps the attended context constant for measurement; otherwise the
    rows start at the sequences' current lengths and the caller moves them with
    :meth:`set_positions` (or :meth:`step_host_full`, which uploads all four input rows).
    """

    def __init__(self, model: MultiLoraModel, seqs, slots, fixed_pos: int | None = None):
        self.m = model
        dev = model.device
        B = len(seqs)
        self.B = B
        pos = [fixed_pos if fixed_pos is not None else model.seq_len[s] for s in seqs]
        self.inp = torch.tensor([[0] * B, pos, list(seqs), list(slots)], dtype=torch.int32,
                                device=dev)
        self.tok, self.pos, self.seq, self.slot = (self.inp[i] for i in range(4))
        self.next_tok = torch.zeros(B, dtype=torch.int32, device=dev)
        # pinned host staging for the end-to-end path (inputs in, sampled tokens out)
        self.h_in = torch.zeros((4, B), dtype=torch.int32).pin_memory()
        self.h_out = torch.zeros(B, dtype=torch.int32).pin_memory()
        self.graph = None
        self.logits = None
        self.kernels_per_step = 0

    def _step(self):
        self.logits = self.m.forward(self.tok, self.pos, self.seq, self.slot, decode=True)
        ops.argmax(self.next_tok, self.logits)

    def capture(self, warmup: int = 2):
        s = torch.cuda.Stream(device=self.m.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self._step()
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        before = ops.launch_count()
        with torch.cuda.graph(self.graph):
            self._step()
        self.kernels_per_step = ops.launch_count() - before
        return self

    def replay(self):
        self.graph.replay()
        return self.next_tok

    def feed_back(self):
        """Device-side: next step's input tokens are this step's argmax."""
        self.tok.copy_(self.next_tok)

    def set_positions(self, pos) -> None:
        """Device positions of the rows for the next replay (host list / array)."""
        self.pos.copy_(torch.as_tensor(np.asarray(pos, dtype=np.int32)), non_blocking=False)

    def step_host(self, tokens: np.ndarray, slots: np.ndarray) -> np.ndarray:
        """End-to-end step through host buffers: H2D tokens+slots, replay, D2H tokens."""
        self.h_in[0].numpy()[:] = tokens
        self.h_in[3].numpy()[:] = slots
        self.tok.copy_(self.h_in[0], non_blocking=True)
        self.slot.copy_(self.h_in[3], non_blocking=True)
        self.graph.replay()
        self.h_out.copy_(self.next_tok, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.h_out.numpy()

    def step_host_full(self, tokens, pos, seqs, slots) -> np.ndarray:
        """End-to-end step with all four input rows from the host: ONE pinned H2D copy,
        replay, ONE D2H copy of the sampled tokens."""
        h = self.h_in.numpy()
        h[0], h[1], h[2], h[3] = tokens, pos, seqs, slots
        self.inp.copy_(self.h_in, non_blocking=True)
        self.graph.replay()
        self.h_out.copy_(self.next_tok, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.h_out.numpy()

    def h2d_bytes(self) -> int:
        return 2 * self.B * 4

    def d2h_bytes(self) -> int:
        return self.B * 4


class DecodeBuckets:
    """Captured decode graphs for batch sizes ``buckets`` (captured on first use).  Spare rows
    of a bucket decode a reserved padding sequence slot at position 0 without an adapter;
    their KV append only ever touches that slot."""

    def __init__(self, model: MultiLoraModel, pad_seq: int, buckets=(1, 2, 4, 8, 16, 32, 64, 96, 128)):
        self.m = model
        self.pad_seq = pad_seq
        self.buckets = tuple(sorted(b for b in buckets if b <= model.max_tokens))
        self.graphs: dict = {}

    def warm(self) -> None:
        """Capture every bucket's graph now (not inside a timed serving step)."""
        for b in self.buckets:
            if b not in self.graphs:
                self.graphs[b] = DecodeGraph(self.m, [self.pad_seq] * b, [-1] * b, fixed_pos=0).capture()

    def bucket(self, n: int) -> int | None:
        for b in self.buckets:
            if b >= n:
                return b
        return None

    def step(self, tokens, pos, seqs, slots) -> np.ndarray | None:
        """Decode ``n`` rows through the smallest bucket >= n; returns the n sampled tokens,
        or None when n exceeds the largest bucket (the caller runs an eager step)."""
        n = len(tokens)
        b = self.bucket(n)
        if b is None:
            return None
        g = self.graphs.get(b)
        if g is None:
            g = DecodeGraph(self.m, [self.pad_seq] * b, [-1] * b, fixed_pos=0).capture()
            self.graphs[b] = g
        pad = b - n
        out = g.step_host_full(np.concatenate([tokens, np.zeros(pad, np.int32)]),
                               np.concatenate([pos, np.zeros(pad, np.int32)]),
                               np.concatenate([seqs, np.full(pad, self.pad_seq, np.int32)]),
                               np.concatenate([slots, np.full(pad, -1, np.int32)]))
        return out[:n].copy()
