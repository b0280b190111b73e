"""Wire formats of a serving frontend (§8 f4): the reference's trace CSV in, request CSV out.

* Trace CSV (``/root/reference/pkg/src/slorasim/workload.py:30,259-282``): header
  ``function_id,arrival_ms,prompt_tokens,output_tokens``; records sorted by (arrival,
  function id); a missing column raises ``ConfigError`` — same reader/writer semantics.
* Request CSV (``metrics.py:217-236``): one row per finished request with TTFT, TPOT, E2E and
  the five cold-start components, numbers formatted ``%.6g`` like the reference; TPOT of a
  one-token request is NaN (``engine.py:111-115``).
* ``replay`` drives a ``ServingRuntime`` from a trace in real time (arrival offsets from the
  start of the replay, optionally time-scaled), with seeded synthetic prompt tokens of each
  record's length — the real-hardware counterpart of ``engine.run`` on a trace.
"""

from __future__ import annotations

import csv
import math
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .spec import ConfigError

TRACE_HEADER = ["function_id", "arrival_ms", "prompt_tokens", "output_tokens"]
REQUEST_CSV_COLUMNS = [
    "request_id", "function", "arrival_ms", "ttft_ms", "tpot_ms", "e2e_ms",
    "cold_container_init_ms", "cold_library_load_ms", "cold_backbone_load_ms",
    "cold_adapter_load_ms", "cold_kernel_compile_ms",
]
COLD_KEYS = ("container_init", "library_load", "backbone_load", "adapter_load", "kernel_compile")


@dataclass(frozen=True)
class TraceRecord:
    function_id: str
    arrival_ms: float
    prompt_tokens: int
    output_tokens: int


def read_trace_csv(path) -> list:
    path = Path(path)
    with open(path, newline="", encoding="utf-8") as fh:
        rd = csv.DictReader(fh)
        missing = set(TRACE_HEADER) - set(rd.fieldnames or [])
        if missing:
            raise ConfigError(f"{path}: missing trace columns {sorted(missing)}")
        recs = [TraceRecord(row["function_id"], float(row["arrival_ms"]), int(row["prompt_tokens"]),
                            int(row["output_tokens"])) for row in rd]
    return sorted(recs, key=lambda r: (r.arrival_ms, r.function_id))


def write_trace_csv(records, path) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_HEADER)
        for r in records:
            a = float(r.arrival_ms)
            w.writerow([r.function_id, int(a) if a.is_integer() else a, r.prompt_tokens, r.output_tokens])


def _fmt(v) -> str:
    return f"{v:.6g}" if isinstance(v, float) else str(v)


def request_row(r, cold: dict | None = None) -> list:
    """Request CSV row of a finished runtime request (``segments.Request``)."""
    ttft = r.first_token_ms - r.arrival_ms
    e2e = r.done_ms - r.arrival_ms
    n = len(r.generated)
    tpot = (r.done_ms - r.first_token_ms) / (n - 1) if n > 1 else math.nan
    cold = cold or {}
    return [r.request_id, r.function_id, _fmt(float(r.arrival_ms)), _fmt(float(ttft)),
            _fmt(float(tpot)), _fmt(float(e2e))] + [_fmt(float(cold.get(k, 0.0))) for k in COLD_KEYS]


def write_requests_csv(requests, path, cold: dict | None = None) -> None:
    """``cold``: optional request_id -> {cold-start component: ms}."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(REQUEST_CSV_COLUMNS)
        for r in requests:
            w.writerow(request_row(r, (cold or {}).get(r.request_id)))


def replay(runtime, records, vocab: int, seed: int = 0, time_scale: float = 1.0,
           max_ctx: int | None = None) -> list:
    """Submit each record when the runtime clock reaches ``arrival_ms * time_scale`` (relative to
    the call), stepping the runtime in between; returns the finished requests.  Prompts are
    seeded random token ids of the record's length (clipped so prompt + output fits
    ``max_ctx``)."""
    rng = np.random.default_rng(seed)
    recs = sorted(records, key=lambda r: (r.arrival_ms, r.function_id))
    t0 = runtime.now_ms()
    i = 0
    while i < len(recs) or runtime.pending():
        now = runtime.now_ms() - t0
        while i < len(recs) and recs[i].arrival_ms * time_scale <= now:
            r = recs[i]
            n_out = max(1, int(r.output_tokens))
            n_in = max(1, int(r.prompt_tokens))
            if max_ctx is not None:
                n_out = min(n_out, max_ctx // 2)
                n_in = min(n_in, max_ctx - n_out)
            prompt = rng.integers(1, vocab, size=n_in).tolist()
            runtime.submit(i, r.function_id, prompt, n_out, arrival_ms=t0 + r.arrival_ms * time_scale)
            i += 1
        if runtime.pending():
            runtime.step()
        else:
            time.sleep(0.0002)
    return runtime.run_until_idle()
