"""Serving runtime for one GPU: batcher rounds -> merged mixed-adapter prefill -> merged decode.

Replaces, on real hardware, the reference engine's modelled path for one GPU:
``_on_scheduler_tick`` -> ``schedule_round`` (``engine.py:607-656``), ``_try_dispatch``'s
``prefill_work_ms = predict_ttft(fn, b)`` (``engine.py:832``), processor-shared prefill and the
``decode_ms_per_token * M`` token loop (``engine.py:259-278,855-910``).  Every round, all
flushed batches on this GPU run as ONE segmented prefill and every active sequence of every
function advances in ONE decode step (the B200 replacement for processor sharing).
Timestamps are real (``time.perf_counter``), after a device synchronize per step.
"""

from __future__ import annotations

import time

import torch

from .batching import BatchQueue, max_batch_size, schedule_round
from .model import MultiLoraModel
from .segments import Request, build_decode, build_prefill


class ServingRuntime:
    def __init__(self, model: MultiLoraModel, functions: dict, gpu_id: str = "gpu0",
                 tick_ms: float = 10.0):
        """``functions``: function_id -> (FunctionSpec-like, adapter slot or -1)."""
        self.m = model
        self.gpu_id = gpu_id
        self.tick_ms = tick_ms
        self.functions = dict(functions)
        self.queues = {fid: BatchQueue(spec, gpu_id, max_batch_size(spec))
                       for fid, (spec, _) in self.functions.items()}
        self.requests: dict = {}
        self.active: list = []
        self.finished: list = []
        self.t0 = time.perf_counter()

    def now_ms(self) -> float:
        return (time.perf_counter() - self.t0) * 1000.0

    def submit(self, request_id, function_id: str, prompt, max_new_tokens: int,
               arrival_ms: float | None = None) -> None:
        """Queue a request (``arrival_ms``: its arrival on this runtime's clock; now if None)."""
        if function_id not in self.functions:
            raise KeyError(f"unknown function {function_id!r}")
        r = Request(request_id, function_id, list(prompt), int(max_new_tokens),
                    self.now_ms() if arrival_ms is None else float(arrival_ms))
        r.adapter_slot = self.functions[function_id][1]
        self.requests[request_id] = r
        self.queues[function_id].enqueue(request_id, r.arrival_ms)

    def _i32(self, a):
        return torch.from_numpy(a).to(self.m.device, non_blocking=True)

    def step(self) -> list:
        """One scheduler tick: flush, prefill the flushed requests together, decode everyone.
        Returns the FlushDecisions taken this round."""
        now = self.now_ms()
        contention = {self.gpu_id: 1 if self.active else 0}
        decisions = schedule_round(list(self.queues.values()), contention, now, self.tick_ms)
        flushed = [self.requests[rid] for d in decisions for rid in d.request_ids]
        if flushed:
            for r in flushed:
                r.seq = self.m.alloc_seq()
            batch = build_prefill(flushed, self.m.seq_len)
            logits = self.m.forward(self._i32(batch.tokens), self._i32(batch.pos),
                                    self._i32(batch.seq), self._i32(batch.slot),
                                    torch.from_numpy(batch.logit_rows).to(self.m.device),
                                    segments=self.m.segments_of(batch.pos, batch.seq))
            for r in batch.requests:
                self.m.seq_len[r.seq] += len(r.prompt)
            nxt = self.m.argmax(logits).cpu().tolist()
            t = self.now_ms()
            for r, tok in zip(batch.requests, nxt):
                r.generated.append(int(tok))
                r.first_token_ms = t
            self.active += batch.requests
        self._retire()
        if self.active:
            batch = build_decode(self.active, self.m.seq_len)
            logits = self.m.forward(self._i32(batch.tokens), self._i32(batch.pos),
                                    self._i32(batch.seq), self._i32(batch.slot), decode=True)
            for r in batch.requests:
                self.m.seq_len[r.seq] += 1
            nxt = self.m.argmax(logits).cpu().tolist()
            for r, tok in zip(batch.requests, nxt):
                r.generated.append(int(tok))
            self._retire()
        return decisions

    def _retire(self) -> None:
        keep = []
        t = self.now_ms()
        for r in self.active:
            if r.done:
                r.done_ms = t
                self.m.free_seq(r.seq)
                self.finished.append(r)
            else:
                keep.append(r)
        self.active = keep

    def pending(self) -> int:
        return sum(q.n for q in self.queues.values()) + len(self.active)

    def run_until_idle(self, max_steps: int = 100000) -> list:
        for _ in range(max_steps):
            if not self.pending():
                break
            self.step()
        torch.cuda.synchronize(self.m.device)
        return self.finished
