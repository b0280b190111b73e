"""Decode engine: one CUDA-graph-captured mixed-adapter decode step per GPU.

The reference advances every co-running batch by ``decode_ms_per_token * M`` per
token (``/root/reference/pkg/src/slorasim/engine.py:888,909``, processor sharing
``engine.py:259-278``).  Here all sequences resident on a GPU — whatever function
(adapter) they belong to — advance together in ONE step: embedding, 32 layers of
tcgen05 GEMMs + multi-LoRA + attention, lm_head and argmax, replayed as a single
CUDA graph so the ~400 kernel launches cost one graph launch.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops
from .model import MultiLoraModel


class LaunchCounter:
    """Counts our C-ABI kernel launches issued through ``ops`` (for gpu_launches)."""

    def __init__(self):
        self.n = 0


class DecodeGraph:
    """Static-shape decode step for ``len(seqs)`` sequences.

    ``fixed_pos``: if given, every replay decodes at this position (KV rewinds), which
    keeps the attended context constant for measurement; otherwise the caller advances
    ``pos`` between replays with :meth:`set_positions`.
    """

    def __init__(self, model: MultiLoraModel, seqs, slots, fixed_pos: int | None = None):
        self.m = model
        dev = model.device
        B = len(seqs)
        self.B = B
        self.tok = torch.zeros(B, dtype=torch.int32, device=dev)
        self.seq = torch.tensor(list(seqs), dtype=torch.int32, device=dev)
        self.slot = torch.tensor(list(slots), dtype=torch.int32, device=dev)
        pos = [fixed_pos if fixed_pos is not None else model.seq_len[s] for s in seqs]
        self.pos = torch.tensor(pos, dtype=torch.int32, device=dev)
        self.next_tok = torch.zeros(B, dtype=torch.int32, device=dev)
        # pinned host staging for the end-to-end path (inputs in, sampled tokens out)
        self.h_in = torch.zeros((2, B), dtype=torch.int32).pin_memory()
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

    def step_host(self, tokens: np.ndarray, slots: np.ndarray) -> np.ndarray:
        """End-to-end step through host buffers: H2D tokens+slots, replay, D2H tokens."""
        self.h_in[0].numpy()[:] = tokens
        self.h_in[1].numpy()[:] = slots
        self.tok.copy_(self.h_in[0], non_blocking=True)
        self.slot.copy_(self.h_in[1], non_blocking=True)
        self.graph.replay()
        self.h_out.copy_(self.next_tok, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.h_out.numpy()

    def h2d_bytes(self) -> int:
        return 2 * self.B * 4

    def d2h_bytes(self) -> int:
        return self.B * 4
