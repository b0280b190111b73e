"""In-graph timeline of a captured decode step (measurement support for bench.py / tools).

Launches of the GEMM (``gemm_sk_kernel``), decode-attention and fused-RMSNorm kernels record
``%globaltimer`` stamps per CTA into a device buffer while ``slx_debug_gemm_trace`` is armed
(one 4096-slot window per launch, the launch's kind in the last slot).  A graph captured in
that state replays with the stamps on, so the timeline is the step as the graph runs it — PDL
overlap included, no events between launches.  The time a launch costs the step is its
exit-to-exit span: from the previous launch's last CTA exit to its own.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

KINDS = {1: "gemm", 2: "gemm", 3: "gemm", 4: "gemm", 5: "attention", 6: "rmsnorm"}
WINDOW = 4096


def trace_graph(make_graph, n_windows: int = 1024, replays: int = 3):
    """Capture ``make_graph()`` (an object with capture()/replay()) with the trace armed, replay
    it, and return the traced launches of the LAST capture pass as
    [(kind, entry_ns, first_data_ns, exit_ns, n_ctas)] in launch order."""
    lib = _lib.load()
    buf = torch.zeros(n_windows * WINDOW, dtype=torch.int64, device="cuda")
    lib.slx_debug_gemm_trace(buf.data_ptr())
    try:
        g = make_graph()
        g.capture(warmup=0)
    finally:
        lib.slx_debug_gemm_trace(None)
    for _ in range(replays):
        g.replay()
    torch.cuda.synchronize()
    t = buf.view(n_windows, WINDOW).cpu().numpy()
    rows = []
    for i in range(n_windows):
        kind = int(t[i, WINDOW - 1] & 0xffffffff)
        if kind == 0:
            continue
        st = t[i, :WINDOW - 16].reshape(-1, 16)
        st = st[st[:, 0] > 0]
        if len(st) == 0:
            continue
        entry = int(st[:, 0].min())
        if kind == 6:
            ex = int(st[:, 7].max())
            first = int(st[:, 2].max())
        else:
            ex = int(max(st[:, 7].max(), st[:, 8].max()))
            col = st[:, 3 if kind != 5 else 2]
            first = int(col[col > 0].min()) if (col > 0).any() else entry
        rows.append((KINDS.get(kind, str(kind)), entry, first, ex, len(st)))
    del g
    return rows


def exit_to_exit(rows) -> dict:
    """Per kind: (launches, total exit-to-exit us) over consecutive traced launches."""
    out: dict = {}
    for i in range(1, len(rows)):
        k = rows[i][0]
        d = out.setdefault(k, [0, 0.0])
        d[0] += 1
        d[1] += (rows[i][3] - rows[i - 1][3]) / 1000.0
    return {k: (n, us) for k, (n, us) in out.items()}


def step_span_us(rows) -> float:
    return (rows[-1][3] - rows[0][1]) / 1000.0 if rows else 0.0


def per_launch(rows, kind: str) -> np.ndarray:
    """Exit-to-exit durations (us) of every launch of ``kind`` (first traced launch excluded)."""
    return np.array([(rows[i][3] - rows[i - 1][3]) / 1000.0 for i in range(1, len(rows))
                     if rows[i][0] == kind])
