"""Calibration bridge (§8 row a1): measure a function's latency law on the B200 runtime.

The reference reduces the whole multi-LoRA forward to four numbers per function
(``FunctionSpec`` fields, ``/root/reference/pkg/src/slorasim/core.py:81-101``; bundled values
``profiles.py:30-36,89-95``): ``prefill_base_ms`` T0 and ``prefill_marginal_ms`` alpha of
``predict_ttft(b) = T0 + alpha*(b-1)`` (``batching.py:17-21``), ``decode_ms_per_token`` and
``kv_cache_bytes_per_request``.  ``profile_function_spec`` measures them with the real
kernels (CUDA events, median of repetitions) so the unchanged batcher/simulator consumes
B200 numbers: T0/alpha from a least-squares fit of mixed-batch prefill time over batch sizes,
decode ms/token from a decode step, KV bytes from the pool layout, SLO = slo_factor * T0
(5x warm prefill).
"""

from __future__ import annotations

import numpy as np
import torch

from .spec import ArtifactKind, ArtifactSpec, FunctionSpec


def _time_ms(fn, reps: int = 5) -> float:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def measure_prefill_ms(model, adapter_slot: int, b: int, prompt_len: int, seed: int = 0) -> float:
    """Time one mixed prefill of ``b`` prompts of ``prompt_len`` tokens (KV pool reused)."""
    rng = np.random.default_rng(seed)
    dev = model.device
    T = b * prompt_len
    toks = torch.from_numpy(rng.integers(1, model.cfg.vocab, size=T).astype(np.int32)).to(dev)
    pos = torch.from_numpy(np.tile(np.arange(prompt_len, dtype=np.int32), b)).to(dev)
    seq = torch.from_numpy(np.repeat(np.arange(b, dtype=np.int32), prompt_len)).to(dev)
    slot = torch.full((T,), adapter_slot, dtype=torch.int32, device=dev)
    last = torch.from_numpy((np.arange(b) + 1) * prompt_len - 1).to(dev)
    segs = [(i * prompt_len, prompt_len, i, 0) for i in range(b)]
    return _time_ms(lambda: model.forward(toks, pos, seq, slot, last, segments=segs))


def measure_decode_ms(model, adapter_slot: int, b: int, ctx: int) -> float:
    """One merged decode step of ``b`` sequences at context ``ctx`` as the serving runtime runs
    it: a captured CUDA graph (engine.DecodeGraph, as runtime.DecodeBuckets replays) when the
    model has the graph-capturable bf16 decode path, else the eager forward."""
    from .engine import DecodeGraph

    dev = model.device
    if model.dtype == torch.bfloat16 and len(model.free_seqs) >= b:
        seqs = [model.alloc_seq() for _ in range(b)]
        try:
            dg = DecodeGraph(model, seqs, [adapter_slot] * b, fixed_pos=ctx)
            dg.capture()
            return _time_ms(dg.replay)
        finally:
            for s_ in seqs:
                model.free_seq(s_)
    toks = torch.ones(b, dtype=torch.int32, device=dev)
    pos = torch.full((b,), ctx, dtype=torch.int32, device=dev)
    seq = torch.arange(b, dtype=torch.int32, device=dev)
    slot = torch.full((b,), adapter_slot, dtype=torch.int32, device=dev)
    return _time_ms(lambda: model.forward(toks, pos, seq, slot, decode=True))


def fit_latency_law(batch_sizes, times_ms) -> tuple[float, float]:
    """Least-squares T(b) = T0 + alpha*(b-1); alpha clamped at >= 0."""
    b = np.asarray(batch_sizes, dtype=np.float64) - 1.0
    t = np.asarray(times_ms, dtype=np.float64)
    A = np.stack([np.ones_like(b), b], 1)
    (t0, alpha), *_ = np.linalg.lstsq(A, t, rcond=None)
    alpha = max(0.0, float(alpha))
    t0 = float(t0) if t0 > 0 else float(t.min())
    return t0, alpha


def profile_function_spec(model, function_id: str, adapter_slot: int, *,
                          backbone_id: str | None = None, prompt_len: int = 60,
                          max_new_tokens: int = 32, batch_sizes=(1, 2, 4, 8),
                          decode_batch: int = 1, slo_factor: float = 5.0,
                          adapter_load_ms: float | None = None, adapter_bytes: int | None = None,
                          backbone_load_ms: float | None = None, container_init_ms: float = 0.0):
    """Measured FunctionSpec for one LoRA function served by ``model`` (needs
    ``model.max_seqs >= max(batch_sizes)`` and ``max_ctx > prompt_len``)."""
    times = [measure_prefill_ms(model, adapter_slot, b, prompt_len) for b in batch_sizes]
    t0, alpha = fit_latency_law(batch_sizes, times)
    decode = measure_decode_ms(model, adapter_slot, decode_batch, prompt_len)
    # the pool reserves max_ctx positions per sequence slot (MultiLoraModel.memory_ledger's
    # kv_slot_bytes), whatever the request's length: that is what admission must book
    kv = model.cfg.kv_bytes_per_token() * model.max_ctx
    if model.dtype == torch.float32:
        kv *= 2
    arts = []
    if backbone_id is None:
        size = model.backbone_bytes()
        ms = backbone_load_ms if backbone_load_ms is not None else 0.0
        arts.append(ArtifactSpec(ArtifactKind.BACKBONE_MODEL, size, ms, ms))
    else:
        size = adapter_bytes or 1
        ms = adapter_load_ms if adapter_load_ms is not None else 0.0
        arts.append(ArtifactSpec(ArtifactKind.ADAPTER_MODEL, size, ms, ms))
    spec = FunctionSpec(id=function_id, artifacts=tuple(arts), slo_ttft_ms=slo_factor * t0,
                        prefill_base_ms=t0, prefill_marginal_ms=alpha,
                        decode_ms_per_token=decode, kv_cache_bytes_per_request=int(kv),
                        container_init_ms=container_init_ms, backbone_id=backbone_id)
    return spec, {"batch_sizes": list(batch_sizes), "prefill_ms": times, "decode_ms": decode}


def to_reference_spec(spec, slorasim_core):
    """Convert to the reference's own ``slorasim.core.FunctionSpec`` (module passed in, so the
    product never imports the reference)."""
    arts = tuple(slorasim_core.ArtifactSpec(slorasim_core.ArtifactKind(a.kind.value), a.size_bytes,
                                            a.load_cold_ms, a.load_from_container_ms)
                 for a in spec.artifacts)
    return slorasim_core.FunctionSpec(
        id=spec.id, artifacts=arts, slo_ttft_ms=spec.slo_ttft_ms,
        prefill_base_ms=spec.prefill_base_ms, prefill_marginal_ms=spec.prefill_marginal_ms,
        decode_ms_per_token=spec.decode_ms_per_token,
        kv_cache_bytes_per_request=spec.kv_cache_bytes_per_request,
        container_init_ms=spec.container_init_ms, backbone_id=spec.backbone_id)
