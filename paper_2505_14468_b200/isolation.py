"""Isolation mode (§8 f3): one process per LoRA function over ONE exported backbone.

The paper's isolation-preserving deployment (``PAPER.md:598-611,641-643``) runs every function
in its own process — own CUDA context, own adapter, own KV cache — while the backbone is
loaded once per GPU and shared read-only.  Here the owner process exports the packed backbone
through CUDA IPC (``torch.multiprocessing`` passes ``cudaIpcMemHandle``s of the weights'
allocations; no copy), and each function process adopts it as its own ``MultiLoraModel``
backbone.  There is no cross-function batching in this mode, and the decode-shrink rows
stacked inside the shared q/k/v/o weights are never written by a function process (its LoRA
runs through the separate shrink/expand kernels).  Each process also measures what its CUDA
context costs — the reference's ``context_overhead_bytes`` (473 MB, ``profiles.py:22``,
booked per process by ``ledger.py:108-118``).
"""

from __future__ import annotations

import queue as _queue

import torch
import torch.multiprocessing as mp

from . import ops


def export_backbone(model) -> dict:
    """IPC-shareable view of a bf16 model's backbone (keep ``model`` alive while shared)."""
    if model.dtype != torch.bfloat16:
        raise ValueError("isolation mode shares the packed bf16 backbone")
    w = {}
    for k, t in model.w.items():
        if isinstance(t, ops.PackedWeight):
            w[k] = ("packed", t.data, t.n, t.k)
        else:
            w[k] = ("tensor", t)
    return {"cfg": model.cfg, "w": w}


def adopt_backbone(model, exported: dict) -> None:
    """Use an exported backbone as ``model``'s own (no allocation, no stacked rows)."""
    model.stack = {}
    model.use_stacked_decode = False
    model.pool.on_install = model.pool.on_evict = None
    w = {}
    for k, v in exported["w"].items():
        w[k] = ops.PackedWeight(v[1], v[2], v[3]) if v[0] == "packed" else v[1]
    model.w = w


def _process_gpu_bytes(pid: int) -> int:
    """Device memory NVML books to process ``pid`` (its CUDA context + its own allocations;
    memory it maps through CUDA IPC stays booked to the exporter)."""
    import pynvml
    pynvml.nvmlInit()
    try:
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            for p in pynvml.nvmlDeviceGetComputeRunningProcesses(h):
                if p.pid == pid and p.usedGpuMemory is not None:
                    return int(p.usedGpuMemory)
        return -1
    finally:
        pynvml.nvmlShutdown()


def _worker(function_id, exported, adapter, lora, limits, jobs, results):
    """One function process: adopt the shared backbone, install its adapter in slot 0, serve
    (prompts, n_new) jobs with greedy decoding; reports its allocator and context bytes."""
    import os

    from .model import MultiLoraModel
    try:
        torch.cuda.init()
        base = torch.cuda.memory_stats()["requested_bytes.all.current"]
        m = MultiLoraModel(exported["cfg"], dtype=torch.bfloat16, n_slots=1, **limits)
        adopt_backbone(m, exported)
        m.pool.load(0, adapter, lora)
        torch.cuda.synchronize()
        own = torch.cuda.memory_stats()["requested_bytes.all.current"] - base
        booked = _process_gpu_bytes(os.getpid())
        context = booked - torch.cuda.memory_reserved() if booked >= 0 else -1
        results.put(("ready", function_id, {"context_bytes": context, "own_bytes": own,
                                            "nvml_process_bytes": booked,
                                            "shared_backbone_bytes": m.backbone_bytes()}))
        while True:
            job = jobs.get()
            if job is None:
                break
            jid, prompts, n_new = job
            seqs, logits = m.prefill(prompts, [0] * len(prompts))
            toks = [m.argmax(logits).cpu().tolist()]
            for _ in range(n_new - 1):
                out = m.decode(seqs, toks[-1], [0] * len(prompts))
                toks.append(m.argmax(out).cpu().tolist())
            for s in seqs:
                m.free_seq(s)
            results.put(("done", function_id, (jid, logits.float().cpu(), toks)))
    except Exception as e:   # surfaced to the owner
        results.put(("error", function_id, repr(e)))


class IsolatedFunctions:
    """The owner side: one spawned process per function, all over ``model``'s backbone."""

    def __init__(self, model, adapters: dict, lora, max_seqs: int = 8, max_ctx: int = 128,
                 max_rank: int = 16, max_tokens: int = 1024, timeout_s: float = 300.0):
        ctx = mp.get_context("spawn")
        self.exported = export_backbone(model)
        self.results = ctx.Queue()
        self.jobs, self.procs, self.info = {}, {}, {}
        self.timeout = timeout_s
        limits = dict(max_seqs=max_seqs, max_ctx=max_ctx, max_rank=max_rank, max_tokens=max_tokens,
                      lora_targets=model.targets)
        for fid, ad in adapters.items():
            q = ctx.Queue()
            p = ctx.Process(target=_worker, args=(fid, self.exported, ad, lora, limits, q, self.results),
                            daemon=True)
            p.start()
            self.jobs[fid], self.procs[fid] = q, p
        for _ in adapters:
            kind, fid, payload = self._get()
            if kind != "ready":
                raise RuntimeError(f"function process {fid}: {payload}")
            self.info[fid] = payload

    def _get(self):
        try:
            return self.results.get(timeout=self.timeout)
        except _queue.Empty:
            raise RuntimeError("function process timed out") from None

    def run(self, function_id: str, prompts, n_new: int):
        """Greedy-generate ``n_new`` tokens for ``prompts`` in the function's own process.
        Returns (prefill logits [n, vocab] fp32, tokens per step)."""
        self.jobs[function_id].put((0, prompts, n_new))
        kind, fid, payload = self._get()
        if kind != "done":
            raise RuntimeError(f"function process {fid}: {payload}")
        _, logits, toks = payload
        return logits, toks

    def close(self) -> None:
        for q in self.jobs.values():
            q.put(None)
        for p in self.procs.values():
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
        torch.cuda.ipc_collect()   # release the exported blocks the children have dropped
