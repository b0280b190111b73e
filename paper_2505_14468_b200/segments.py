"""Segment builder: one scheduler round's FlushDecisions -> one adapter-segmented mixed batch.

The reference dispatches every ``FlushDecision`` (``batching.py:99-105``) as its own batch and
lets M co-running batches share the GPU by processor sharing (``engine.py:259-278``).  On the
B200 all flushes of a round that target the same GPU/backbone become ONE token-major batch:
each request is a contiguous segment carrying its function's adapter slot, which is exactly
the input of the SGMV prefill (``seg_indptr``/``seg_slot``) and, one token per sequence, of
the BGMV decode (per-token slot).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Request:
    request_id: object
    function_id: str
    prompt: list
    max_new_tokens: int
    arrival_ms: float = 0.0
    # filled by the runtime
    seq: int = -1
    adapter_slot: int = -1
    generated: list = field(default_factory=list)
    first_token_ms: float | None = None
    done_ms: float | None = None

    @property
    def done(self) -> bool:
        return len(self.generated) >= self.max_new_tokens


@dataclass
class MixedBatch:
    """Token-major batch: per-token arrays plus the per-request segment structure."""

    requests: list
    tokens: np.ndarray      # int32 [T]
    pos: np.ndarray         # int32 [T]
    seq: np.ndarray         # int32 [T]  KV-pool sequence slot
    slot: np.ndarray        # int32 [T]  adapter slot (-1 = backbone only)
    seg_indptr: np.ndarray  # int32 [S+1] request segments
    seg_slot: np.ndarray    # int32 [S]
    logit_rows: np.ndarray  # int64 [S] last token of each segment

    @property
    def n_tokens(self) -> int:
        return int(self.tokens.size)


def build_prefill(requests: list, seq_len: list) -> MixedBatch:
    """Prefill segments, requests grouped by adapter slot (stable), each request continuing
    its KV sequence at ``seq_len[req.seq]``."""
    order = sorted(requests, key=lambda r: (r.adapter_slot, str(r.function_id)))
    toks, pos, sq, sl, indptr, seg_slot, last = [], [], [], [], [0], [], []
    for r in order:
        L = len(r.prompt)
        if L == 0:
            raise ValueError(f"request {r.request_id}: empty prompt")
        start = seq_len[r.seq]
        toks += list(r.prompt)
        pos += list(range(start, start + L))
        sq += [r.seq] * L
        sl += [r.adapter_slot] * L
        indptr.append(indptr[-1] + L)
        seg_slot.append(r.adapter_slot)
        last.append(indptr[-1] - 1)
    i32 = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
    return MixedBatch(order, i32(toks), i32(pos), i32(sq), i32(sl), i32(indptr), i32(seg_slot),
                      np.asarray(last, dtype=np.int64))


def build_decode(requests: list, seq_len: list) -> MixedBatch:
    """One token per active sequence (its last generated token) at its next position."""
    i32 = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
    n = len(requests)
    return MixedBatch(list(requests), i32([r.generated[-1] for r in requests]),
                      i32([seq_len[r.seq] for r in requests]), i32([r.seq for r in requests]),
                      i32([r.adapter_slot for r in requests]), i32(np.arange(n + 1)),
                      i32([r.adapter_slot for r in requests]), np.arange(n, dtype=np.int64))


def build_mixed(prefill: list, decode: list, seq_len: list) -> tuple[MixedBatch, int]:
    """One forward for a round with both new prompts and running sequences: the prefill
    segments followed by one 1-token segment per running sequence (its last generated token
    at its next position, a segment with a cached prefix).  Returns the batch and the number
    of prefill requests (``batch.requests[:n]``; the rest are the decode rows)."""
    p = build_prefill(prefill, seq_len)
    d = build_decode(decode, seq_len)
    T = p.n_tokens
    cat = np.concatenate
    return MixedBatch(p.requests + d.requests, cat([p.tokens, d.tokens]), cat([p.pos, d.pos]),
                      cat([p.seq, d.seq]), cat([p.slot, d.slot]),
                      cat([p.seg_indptr, d.seg_indptr[1:] + T]).astype(np.int32),
                      cat([p.seg_slot, d.seg_slot]),
                      cat([p.logit_rows, d.logit_rows + T])), len(p.requests)


def group_by_gpu(decisions) -> dict:
    """FlushDecisions of one round grouped per target GPU (one mixed batch each)."""
    out: dict = {}
    for d in decisions:
        out.setdefault(d.gpu_id, []).append(d)
    return out
