"""torch-tensor front end of the C ABI (device memory and streams come from PyTorch).

Every function enqueues on ``torch.cuda.current_stream()`` and never synchronises,
so a sequence of calls can be captured into a CUDA graph.  Shapes and dtypes are
validated here (ValueError) and again in C (status codes).
"""

from __future__ import annotations

import ctypes

import numpy as np

import torch

from . import _lib
from ._lib import (DT_BF16, DT_F32, EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL, W_ROWMAJOR, W_TILED,
                   GemmTuning, L2Prefetch, LoraDelta, LoraTarget, RopeKV, SplitKIn, check)

_DT = {torch.bfloat16: DT_BF16, torch.float32: DT_F32}

# ------------------------------------------------------------------ launch accounting / timing
_LAUNCHES = 0
_TIMER = None   # optional KernelTimer: CUDA events around every op, by category


def launch_count() -> int:
    """Number of libslora_b200 kernel launches issued through this module so far."""
    return _LAUNCHES


class KernelTimer:
    """Records a CUDA event pair around each op on the current stream; durations are read
    after a synchronize.  Used by bench.py for per-kernel-class roofline numbers."""

    def __init__(self):
        self.records = []   # (category, start_event, end_event, meta)

    def __enter__(self):
        global _TIMER
        _TIMER = self
        return self

    def __exit__(self, *exc):
        global _TIMER
        _TIMER = None

    def durations(self):
        out = {}
        for cat, a, b, meta in self.records:
            ms, n, metas = out.get(cat, (0.0, 0, []))
            out[cat] = (ms + a.elapsed_time(b), n + 1, metas + [meta])
        return out


def _op(category: str, n_launch: int = 1):
    def deco(fn):
        def wrapped(*args, **kwargs):
            global _LAUNCHES
            _LAUNCHES += n_launch
            if _TIMER is None:
                return fn(*args, **kwargs)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn(*args, **kwargs)
            b.record()
            meta = tuple(tuple(x.shape) for x in args if isinstance(x, torch.Tensor))
            _TIMER.records.append((category, a, b, meta))
            return out
        wrapped.__name__ = fn.__name__
        wrapped.__doc__ = fn.__doc__
        return wrapped
    return deco


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported activation dtype {t.dtype}") from None


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("expected a row-major 2-D tensor with unit column stride")
    return t.stride(0)


class Workspace:
    """Zero-initialised device scratch (counters inside must start at zero; kernels keep
    them zero).  Grows only outside graph capture."""

    def __init__(self, device, nbytes: int = 64 << 20):
        self.device = torch.device(device)
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)

    def get(self, nbytes: int) -> torch.Tensor:
        if nbytes > self.buf.numel():
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError("workspace growth during CUDA graph capture")
            self.buf = torch.zeros(max(nbytes, 2 * self.buf.numel()), dtype=torch.uint8,
                                   device=self.device)
        return self.buf


_DEFAULT_WS: dict = {}


def default_workspace(device) -> "Workspace":
    """Per-device zeroed GEMM workspace (split-K partials + self-cleaning counters), sized
    once so it never grows during CUDA graph capture.  One stream at a time may use it."""
    d = torch.device(device)
    if d not in _DEFAULT_WS:
        _DEFAULT_WS[d] = Workspace(d, 48 << 20)
    return _DEFAULT_WS[d]


# ---------------------------------------------------------------------------------- K1
class PackedWeight:
    """bf16 W[N, K] packed in the SLX_W_TILED layout ([N/128][K/64][128][64], zero-padded):
    every TMA box the GEMM loads is one contiguous 16 KB HBM burst.  ``n_extra`` rows after
    the first ``n`` hold the stacked LoRA A of every adapter slot (decode shrink rows)."""

    def __init__(self, data: torch.Tensor, n: int, k: int, n_extra: int = 0):
        self.data, self.n, self.k, self.n_extra = data, n, k, n_extra
        self.shape = (n, k)
        self.dtype = torch.bfloat16

    def numel(self) -> int:
        return self.n * self.k

    def element_size(self) -> int:
        return 2


@_op("pack", 1)
def pack_weight(w: torch.Tensor, extra_rows: int = 0) -> PackedWeight:
    if w.dtype != torch.bfloat16 or w.dim() != 2 or w.stride(1) != 1:
        raise ValueError("pack_weight: bf16 row-major [N, K] expected")
    N, K = w.shape
    lib = _lib.load()
    if extra_rows:
        if N % 128:
            raise ValueError("pack_weight: stacked rows need N % 128 == 0")
        out = torch.zeros(lib.slx_packed_weight_elems(N + extra_rows, K), dtype=torch.bfloat16,
                          device=w.device)
        check(lib.slx_pack_weight_rows(_ptr(out), _ptr(w), N, K, w.stride(0), 0, _stream()),
              "slx_pack_weight_rows")
        return PackedWeight(out, N, K, extra_rows)
    out = torch.empty(lib.slx_packed_weight_elems(N, K), dtype=torch.bfloat16, device=w.device)
    check(lib.slx_pack_weight(_ptr(out), _ptr(w), N, K, w.stride(0), _stream()), "slx_pack_weight")
    return PackedWeight(out, N, K)


@_op("pack", 1)
def pack_rows(pw: PackedWeight, src: torch.Tensor | None, n_rows: int, row0: int) -> None:
    """(Re)write rows [row0, row0+n_rows) of a packed weight from row-major bf16 src (None =
    zeros)."""
    if src is not None and (src.dtype != torch.bfloat16 or src.stride(-1) != 1):
        raise ValueError("pack_rows: bf16 row-major src expected")
    ld = src.stride(0) if src is not None and src.dim() == 2 else pw.k
    check(_lib.load().slx_pack_weight_rows(_ptr(pw.data), _ptr(src), n_rows, pw.k, ld, row0,
                                           _stream()), "slx_pack_weight_rows")


def l2_prefetch(*regions) -> L2Prefetch | None:
    """slx_l2_prefetch of up to two (tensor, nbytes) regions the next kernel streams first."""
    regions = [r for r in regions if r is not None and r[1] > 0]
    if not regions:
        return None
    if len(regions) > 2:
        raise ValueError("l2_prefetch: at most two regions")
    pf = L2Prefetch()
    for i, (t, n) in enumerate(regions):
        pf.ptr[i] = t.data_ptr()
        pf.bytes[i] = min(int(n), t.numel() * t.element_size())
    return pf


@_op("gemm", 1)
def gemm(a: torch.Tensor, w, out: torch.Tensor | None = None, *,
         epilogue: int = EPI_NONE, residual: torch.Tensor | None = None,
         out_dtype: torch.dtype | None = None, ws=None, side: torch.Tensor | None = None,
         prefetch: L2Prefetch | None = None, tuning: dict | None = None) -> torch.Tensor:
    """bf16 tcgen05 GEMM: out = a @ w.T (+ residual | silu*mul of blocked gate/up).
    ``w`` is a row-major bf16 [N, K] tensor or a :class:`PackedWeight`; with ``side`` (fp32
    [M, n_extra]) the packed weight's stacked extra rows are computed too (LoRA shrink);
    ``prefetch`` (l2_prefetch) names the next kernel's first bytes; ``tuning`` (fields of
    slx_gemm_tuning, e.g. ``{"tile_kernel": 1, "splits": 4}``) forces a tiling (tests/tools)."""
    if a.dtype != torch.bfloat16 or w.dtype != torch.bfloat16:
        raise ValueError("gemm: a and w must be bf16")
    M, K = a.shape
    N, Kw = w.shape
    n_main, n_tot = N, N
    if isinstance(w, PackedWeight):
        layout, wt = W_TILED, w.data
        if side is not None:
            if side.dtype != torch.float32 or side.shape[0] != M or side.shape[1] < w.n_extra:
                raise ValueError("gemm: side output must be fp32 [M, n_extra]")
            n_tot = N + w.n_extra
    else:
        if not w.is_contiguous():
            raise ValueError("gemm: w must be contiguous [N, K]")
        layout, wt = W_ROWMAJOR, w
    if Kw != K:
        raise ValueError("gemm: K mismatch")
    n_out = N // 2 if epilogue == EPI_SILU_MUL else N
    if out is None:
        out = torch.empty((M, n_out), dtype=out_dtype or torch.bfloat16, device=a.device)
    if residual is not None and residual.dtype != out.dtype:
        raise ValueError("gemm: residual must have the output dtype")
    wsb = (ws if ws is not None else default_workspace(a.device)).get(
        _lib.load().slx_gemm_workspace_bytes(M, n_tot, K, epilogue))
    tu = None
    if tuning:
        tu = GemmTuning()
        for k, v in tuning.items():
            setattr(tu, k, int(v))
    check(_lib.load().slx_gemm_bf16_ex(_ptr(a), _ld(a), _ptr(wt), _ptr(out), _ld(out), _dt(out),
                                       _ptr(residual), _ld(residual) if residual is not None else 0,
                                       M, n_tot, K, epilogue, layout, n_main,
                                       _ptr(side) if n_tot > n_main else None,
                                       _ld(side) if n_tot > n_main else 0, _ptr(wsb), wsb.numel(),
                                       None if prefetch is None else ctypes.byref(prefetch),
                                       None if tu is None else ctypes.byref(tu),
                                       _stream()), "slx_gemm_bf16")
    return out


@_op("gemm", 1)
def gemm_f32(a: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None, *,
             residual: torch.Tensor | None = None) -> torch.Tensor:
    """fp32-parity GEMM: fp32 activations x bf16 weights (upcast exactly), fp32 out."""
    if a.dtype != torch.float32 or w.dtype != torch.bfloat16:
        raise ValueError("gemm_f32: a fp32, w bf16")
    M, K = a.shape
    N = w.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=a.device)
    epi = EPI_RESIDUAL if residual is not None else EPI_NONE
    check(_lib.load().slx_gemm_f32(_ptr(a), _ld(a), _ptr(w), _ptr(out), _ld(out), _ptr(residual),
                                   _ld(residual) if residual is not None else 0, M, N, K, epi,
                                   _stream()), "slx_gemm_f32")
    return out


# ---------------------------------------------------------------------------------- K2/K3
def sm_count() -> int:
    """SMs of the current device (slx_device_sm_count)."""
    n = ctypes.c_int(0)
    check(_lib.load().slx_device_sm_count(ctypes.byref(n)), "slx_device_sm_count")
    return n.value


def lora_workspace_bytes(n_tok: int, n_slots: int, max_rank: int, n_targets: int) -> int:
    return _lib.load().slx_lora_workspace_bytes(n_tok, n_slots, max_rank, n_targets)


@_op("lora_plan", 1)
def lora_plan_tokens(tok_slot: torch.Tensor, n_slots: int, ws: torch.Tensor) -> None:
    check(_lib.load().slx_lora_plan_tokens(_ptr(tok_slot), tok_slot.numel(), n_slots, _ptr(ws),
                                           ws.numel(), _stream()), "slx_lora_plan_tokens")


@_op("lora_plan", 1)
def lora_plan_segments(seg_indptr: torch.Tensor, seg_slot: torch.Tensor, n_tok: int,
                       n_slots: int, ws: torch.Tensor) -> None:
    check(_lib.load().slx_lora_plan_segments(_ptr(seg_indptr), _ptr(seg_slot), seg_slot.numel(),
                                             n_tok, n_slots, _ptr(ws), ws.numel(), _stream()),
          "slx_lora_plan_segments")


def make_targets(specs) -> ctypes.Array:
    """specs: iterable of (a_ptr_table, b_ptr_table, d_out, col_off, col_blk, col_stride)."""
    specs = list(specs)
    arr = (LoraTarget * len(specs))()
    for i, (a, b, d_out, off, blk, stride) in enumerate(specs):
        arr[i] = LoraTarget(a.data_ptr(), b.data_ptr(), d_out, off, blk, stride)
    return arr


@_op("lora", 2)
def lora_apply(y: torch.Tensor, x: torch.Tensor, d_in: int, slot_rank: torch.Tensor,
               slot_scale: torch.Tensor, max_rank: int, targets, ws: torch.Tensor) -> None:
    """y[t, col(n)] += scale * (x[t, :d_in] A^T) B^T over the plan stored in ws."""
    if y.dtype != x.dtype:
        raise ValueError("lora_apply: x and y dtypes differ")
    check(_lib.load().slx_lora_apply(_dt(y), _ptr(y), _ld(y), _ptr(x), _ld(x), x.shape[0], d_in,
                                     _ptr(slot_rank), _ptr(slot_scale), slot_rank.numel(),
                                     max_rank, len(targets), targets, _ptr(ws), ws.numel(),
                                     _stream()), "slx_lora_apply")


@_op("lora", 3)
def lora_bgmv(y, x, tok_slot, slot_rank, slot_scale, max_rank, targets, ws, d_in=None):
    d_in = x.shape[1] if d_in is None else d_in
    check(_lib.load().slx_lora_bgmv(_dt(y), _ptr(y), _ld(y), _ptr(x), _ld(x), _ptr(tok_slot),
                                    x.shape[0], d_in, _ptr(slot_rank), _ptr(slot_scale),
                                    slot_rank.numel(), max_rank, len(targets), targets, _ptr(ws),
                                    ws.numel(), _stream()), "slx_lora_bgmv")


@_op("lora", 3)
def lora_sgmv(y, x, seg_indptr, seg_slot, slot_rank, slot_scale, max_rank, targets, ws,
              d_in=None):
    d_in = x.shape[1] if d_in is None else d_in
    check(_lib.load().slx_lora_sgmv(_dt(y), _ptr(y), _ld(y), _ptr(x), _ld(x), _ptr(seg_indptr),
                                    _ptr(seg_slot), seg_slot.numel(), x.shape[0], d_in,
                                    _ptr(slot_rank), _ptr(slot_scale), slot_rank.numel(),
                                    max_rank, len(targets), targets, _ptr(ws), ws.numel(),
                                    _stream()), "slx_lora_sgmv")


@_op("lora", 1)
def lora_expand(y: torch.Tensor, v_all: torch.Tensor, slot_rank, slot_scale, max_rank: int,
                targets, v_col_off, ws: torch.Tensor, v_slot_stride: int | None = None) -> None:
    """Decode expand in place: y[t, col(n)] += scale * v . B_slot^T over the plan in ws.  v from
    the GEMM-side stacked shrink (``v_slot_stride`` = max_rank, the default) or from the
    gathered shrink (``v_slot_stride=0``)."""
    offs = (ctypes.c_int * len(v_col_off))(*v_col_off)
    stride = max_rank if v_slot_stride is None else int(v_slot_stride)
    check(_lib.load().slx_lora_expand(_dt(y), _ptr(y), _ld(y), _ptr(v_all), _ld(v_all), y.shape[0],
                                      _ptr(slot_rank), _ptr(slot_scale), slot_rank.numel(), max_rank,
                                      len(targets), targets, offs, stride, _ptr(ws), ws.numel(),
                                      _stream()), "slx_lora_expand")


@_op("lora", 1)
def lora_shrink(v: torch.Tensor, x: torch.Tensor, slot_rank, max_rank: int, targets, v_col_off,
                ws: torch.Tensor) -> None:
    """Gathered decode shrink over the plan in ws: v[t, v_col_off[i] + j] = x_t . A_slot(t)[j]
    (fp32, unscaled) for the adapters present in the batch only."""
    if v.dtype != torch.float32:
        raise ValueError("lora_shrink: v must be fp32")
    offs = (ctypes.c_int * len(v_col_off))(*v_col_off)
    check(_lib.load().slx_lora_shrink(_dt(x), _ptr(v), _ld(v), _ptr(x), _ld(x), x.shape[0],
                                      x.shape[1], _ptr(slot_rank), slot_rank.numel(), max_rank,
                                      len(targets), targets, offs, _ptr(ws), ws.numel(), _stream()),
          "slx_lora_shrink")


GROUP_MAX = 16


def rope_kv(heads, kv_heads, head_dim, tok_pos, tok_seq, cos, sin, k_cache, v_cache) -> RopeKV:
    """slx_rope_kv: fuse RoPE + the KV append into a q/k/v projection (gemm_lorafold)."""
    r = RopeKV()
    r.tok_pos, r.tok_seq = tok_pos.data_ptr(), tok_seq.data_ptr()
    r.cos_tab, r.sin_tab, r.max_pos = cos.data_ptr(), sin.data_ptr(), cos.shape[0]
    r.k_cache, r.v_cache, r.max_ctx = k_cache.data_ptr(), v_cache.data_ptr(), k_cache.shape[2]
    r.heads, r.kv_heads, r.head_dim = heads, kv_heads, head_dim
    return r


@_op("gemm", 1)
def gemm_lorafold(a: torch.Tensor, w, out: torch.Tensor, gtiles: torch.Tensor, v: torch.Tensor,
                  t_bound, b_ptrs, b_rows, ranks, residual: torch.Tensor | None = None,
                  rope: RopeKV | None = None) -> torch.Tensor:
    """Prefill backbone GEMM with the LoRA expand as one extra K block per grouped tile
    (slx_gemm_bf16_lorafold).  w: PackedWeight; v: bf16 [T, 64 * targets] shrink (scale folded);
    b_ptrs: per (adapter, target) B addresses (adapter-major); ``rope`` (rope_kv): RoPE + KV
    append fused into the epilogue (q/k/v projection)."""
    if a.dtype != torch.bfloat16 or not isinstance(w, PackedWeight) or v.dtype != torch.bfloat16:
        raise ValueError("gemm_lorafold: bf16 activations, packed weight, bf16 v")
    M, K = a.shape
    nt = len(t_bound)
    arr = lambda t, vals: (t * len(vals))(*vals)  # noqa: E731
    epi = EPI_RESIDUAL if residual is not None else EPI_NONE
    check(_lib.load().slx_gemm_bf16_lorafold(
        _ptr(a), _ld(a), _ptr(w.data), W_TILED, _ptr(out), _ld(out), _dt(out), _ptr(residual),
        _ld(residual) if residual is not None else 0, M, w.n, K, epi, _ptr(gtiles), gtiles.shape[0],
        _ptr(v), _ld(v), nt, arr(ctypes.c_int, list(t_bound)), len(ranks),
        arr(ctypes.c_uint64, list(b_ptrs)), arr(ctypes.c_int, list(b_rows)),
        arr(ctypes.c_int, list(ranks)), None if rope is None else ctypes.byref(rope), _stream()),
        "slx_gemm_bf16_lorafold")
    return out


@_op("lora", 1)
def gemm_grouped(a: torch.Tensor, k: int, groups, gtiles: torch.Tensor, out: torch.Tensor, n: int,
                 residual: torch.Tensor | None = None, n_seg: int = 1) -> torch.Tensor:
    """Grouped tcgen05 GEMM.  groups: [(w_ptr, w_rows, w_cols, w_ld, alpha)] (<= 16 groups;
    with ``n_seg`` > 1, n_seg entries per group, group-major: output columns [64 s, 64 s + 64)
    from entry s of the tile's group); gtiles: device int32 [n_tiles, 4] of (group, m0, m_rows,
    n0)."""
    g = list(groups)
    if not 1 <= len(g) // n_seg <= GROUP_MAX or len(g) % n_seg:
        raise ValueError("gemm_grouped: 1..16 groups per call (n_seg entries each)")
    arr = lambda t, vals: (t * len(vals))(*vals)  # noqa: E731
    epi = EPI_RESIDUAL if residual is not None else EPI_NONE
    check(_lib.load().slx_gemm_grouped_bf16(
        _ptr(a), _ld(a), a.shape[0], k, len(g) // n_seg, n_seg, arr(ctypes.c_uint64, [x[0] for x in g]),
        arr(ctypes.c_int, [x[1] for x in g]), arr(ctypes.c_int, [x[2] for x in g]),
        arr(ctypes.c_int, [x[3] for x in g]), arr(ctypes.c_float, [x[4] for x in g]),
        _ptr(out), _ld(out), _dt(out), _ptr(residual), _ld(residual) if residual is not None else 0,
        n, epi, _ptr(gtiles), gtiles.shape[0], _stream()), "slx_gemm_grouped_bf16")
    return out


# ---------------------------------------------------------------------------------- K4
@_op("embedding", 1)
def embedding(out, table, tokens):
    check(_lib.load().slx_embedding(_dt(out), _ptr(out), _ptr(table), _ptr(tokens), tokens.numel(),
                                    table.shape[1], table.shape[0], _stream()), "slx_embedding")
    return out


@_op("rmsnorm", 1)
def rmsnorm(out, x, w, eps: float):
    check(_lib.load().slx_rmsnorm(_dt(out), _ptr(out), _ld(out), _ptr(x), _ld(x), _ptr(w),
                                  x.shape[0], w.numel(), float(eps), _stream()), "slx_rmsnorm")
    return out


def make_delta(v_all: torch.Tensor | None, tok_slot, slot_rank, slot_scale, max_rank: int, targets,
               v_slot_stride: int | None = None):
    """slx_lora_delta for a fused decode expand.  targets: [(b_ptr_table, v_col_off, y_col_off,
    d_out)] (<= 4); v_all: the fp32 shrink output [n_tok, ldv], or None when the consumer
    takes v from split-K pieces (v_col_off then counts from the pieces' n_main).
    ``v_slot_stride``: columns between slots' v blocks (default max_rank: the stacked shrink;
    0: a gathered shrink holding only the token's own adapter)."""
    targets = list(targets)
    if not 1 <= len(targets) <= 4 or (v_all is not None and v_all.dtype != torch.float32):
        raise ValueError("make_delta: 1..4 targets and an fp32 v_all")
    d = LoraDelta()
    if v_all is not None:
        d.v, d.ldv = v_all.data_ptr(), _ld(v_all)
    d.tok_slot, d.slot_rank, d.slot_scale = tok_slot.data_ptr(), slot_rank.data_ptr(), slot_scale.data_ptr()
    d.max_rank, d.n_targets = max_rank, len(targets)
    d.v_slot_stride = max_rank if v_slot_stride is None else int(v_slot_stride)
    for i, (b, voff, yoff, dout) in enumerate(targets):
        d.b_ptrs[i], d.v_col_off[i], d.y_col_off[i], d.d_out[i] = b.data_ptr(), voff, yoff, dout
    return d


def splitk_bytes(M: int, N: int, splits: int) -> int:
    return _lib.load().slx_gemm_splitk_bytes(M, N, splits)


@_op("gemm", 1)
def gemm_splitk(a: torch.Tensor, w, splits: int, part: torch.Tensor, prefetch=None) -> SplitKIn:
    """Decode projection as split-K pieces (no epilogue) for the consuming kernel; returns the
    slx_splitk_in describing them.  w: PackedWeight (main + stacked rows)."""
    if a.dtype != torch.bfloat16 or not isinstance(w, PackedWeight):
        raise ValueError("gemm_splitk: bf16 activations and a packed weight")
    M, K = a.shape
    N = w.n + w.n_extra
    check(_lib.load().slx_gemm_bf16_splitk(_ptr(a), _ld(a), _ptr(w.data), M, N, K, splits,
                                           _ptr(part), part.numel() * part.element_size(),
                                           None if prefetch is None else ctypes.byref(prefetch),
                                           _stream()), "slx_gemm_bf16_splitk")
    sk = SplitKIn()
    sk.part, sk.splits, sk.bm, sk.n_main = part.data_ptr(), splits, (M + 15) // 16 * 16, w.n
    return sk


@_op("rmsnorm", 1)
def rmsnorm_fused(out, x, w, eps: float, sk=None, delta=None, prefetch=None):
    """x = round(x + split-K pieces) (the projection's residual epilogue), x += LoRA delta
    (v from the pieces when the delta has no v), out = rmsnorm(x); ``prefetch`` (l2_prefetch):
    the next GEMM's weights, requested at kernel entry."""
    check(_lib.load().slx_rmsnorm_fused(_dt(out), _ptr(out), _ld(out), _ptr(x), _ld(x), _ptr(w),
                                        x.shape[0], w.numel(), float(eps),
                                        None if sk is None else ctypes.byref(sk),
                                        None if delta is None else ctypes.byref(delta),
                                        None if prefetch is None else ctypes.byref(prefetch),
                                        _stream()),
          "slx_rmsnorm_fused")
    return out


@_op("rmsnorm", 1)
def rmsnorm_lora(out, x, w, eps: float, delta):
    """x += LoRA delta (fused o-projection expand, written back), out = rmsnorm(x)."""
    check(_lib.load().slx_rmsnorm_lora(_dt(out), _ptr(out), _ld(out), _ptr(x), _ld(x), _ptr(w),
                                       x.shape[0], w.numel(), float(eps),
                                       None if delta is None else ctypes.byref(delta), _stream()),
          "slx_rmsnorm_lora")
    return out


@_op("rope_kv", 1)
def rope_kv_write(qkv, heads, kv_heads, head_dim, tok_pos, tok_seq, cos, sin, k_cache, v_cache):
    check(_lib.load().slx_rope_kv_write(_dt(qkv), _ptr(qkv), _ld(qkv), qkv.shape[0], heads,
                                        kv_heads, head_dim, _ptr(tok_pos), _ptr(tok_seq),
                                        _ptr(cos), _ptr(sin), cos.shape[0], _ptr(k_cache),
                                        _ptr(v_cache), k_cache.shape[2], _stream()),
          "slx_rope_kv_write")


@_op("attention", 1)
def attention(out, qkv, heads, kv_heads, head_dim, tok_pos, tok_seq, k_cache, v_cache):
    check(_lib.load().slx_attention(_dt(out), _ptr(out), _ld(out), _ptr(qkv), _ld(qkv),
                                    qkv.shape[0], heads, kv_heads, head_dim, _ptr(tok_pos),
                                    _ptr(tok_seq), _ptr(k_cache), _ptr(v_cache), k_cache.shape[2],
                                    _stream()), "slx_attention")
    return out


@_op("attention", 1)
def rope_attention_decode(out, qkv, heads, kv_heads, head_dim, tok_pos, tok_seq, cos, sin,
                          k_cache, v_cache, lora=None, prefetch=None, pool_seqs=None):
    """Decode-step RoPE + KV append + attention in one kernel (each token = next position of
    its own sequence); ``lora`` (make_delta) fuses the q/k/v LoRA expand, ``prefetch``
    (l2_prefetch) names the next kernel's first bytes; ``pool_seqs`` (default: the caches'
    sequence slots) = 0 selects the one-CTA-per-(token, head) kernel (tests)."""
    check(_lib.load().slx_rope_attention_decode(
        _dt(out), _ptr(out), _ld(out), _ptr(qkv), _ld(qkv), qkv.shape[0], heads, kv_heads, head_dim,
        _ptr(tok_pos), _ptr(tok_seq), _ptr(cos), _ptr(sin), cos.shape[0], _ptr(k_cache),
        _ptr(v_cache), k_cache.shape[2], k_cache.shape[0] if pool_seqs is None else int(pool_seqs),
        None if lora is None else ctypes.byref(lora),
        None if prefetch is None else ctypes.byref(prefetch), _stream()),
        "slx_rope_attention_decode")
    return out


def prefill_plan(segments, heads: int, device, bq: int | None = None):
    """[(tok0, n, seq, pos0)] segments -> the flash prefill's tile table (int32 [n_tiles, 4] of
    <= bq queries of one segment) and work items (int32 [n_items, 4] = (tile_a, tile_b, head,
    0)): per segment and head, consecutive tiles are paired (tile_b = the tile before tile_a,
    so its keys are a prefix of a's and both stream the same K/V blocks in one CTA); items are
    ordered by cost (key blocks of both tiles), longest first, so the persistent CTAs' strided
    shares come out even."""
    if bq is None:
        bq = int(_lib.load().slx_flash_prefill_tile_queries())
    # vectorised (a serving round can carry hundreds of segments: decode rows of mixed rounds)
    sg = np.asarray(segments, dtype=np.int64).reshape(-1, 4)
    tok0, n, seq, pos0 = sg[:, 0], sg[:, 1], sg[:, 2], sg[:, 3]
    nt = (n + bq - 1) // bq                       # tiles per segment
    first = np.cumsum(nt) - nt                    # first tile id of each segment
    tseg = np.repeat(np.arange(len(sg)), nt)
    q = (np.arange(int(nt.sum())) - first[tseg]) * bq
    tiles = np.stack([tok0[tseg] + q, np.minimum(bq, n[tseg] - q), seq[tseg], pos0[tseg] + q], 1)
    npair = (nt + 1) // 2                         # pairs (tile_a, tile_b) per segment
    pfirst = np.cumsum(npair) - npair
    pseg = np.repeat(np.arange(len(sg)), npair)
    kk = 2 * (np.arange(int(npair.sum())) - pfirst[pseg])
    has_b = kk + 1 < nt[pseg]
    pa = np.where(has_b, first[pseg] + kk + 1, first[pseg] + kk)
    pb = np.where(has_b, first[pseg] + kk, -1)
    per = heads * npair                           # items per segment: head-major, then pair
    iseg = np.repeat(np.arange(len(sg)), per)
    w = np.arange(int(per.sum())) - (np.cumsum(per) - per)[iseg]
    h = w // npair[iseg]
    pg = pfirst[iseg] + w % npair[iseg]
    a, b = pa[pg], pb[pg]
    ends = tiles[:, 3] + tiles[:, 1]
    cost = -(-ends[a] // 64) + np.where(b >= 0, -(-ends[np.maximum(b, 0)] // 64), 0)
    order = np.argsort(-cost, kind="stable")      # longest first (stable, as list.sort)
    items = np.stack([a, b, h, np.zeros_like(h)], 1)[order]
    t = torch.from_numpy(tiles.astype(np.int32)).reshape(-1, 4)
    it = torch.from_numpy(np.ascontiguousarray(items, dtype=np.int32)).reshape(-1, 4)
    return t.to(device), it.to(device)


@_op("attention", 1)
def attention_prefill(out, qkv, heads, kv_heads, head_dim, plan, k_cache, v_cache):
    """tcgen05 causal flash attention for prefill segments (plan from prefill_plan)."""
    tiles, items = plan
    check(_lib.load().slx_attention_prefill(_ptr(out), _ld(out), _ptr(qkv), _ld(qkv), qkv.shape[0],
                                            heads, kv_heads, head_dim, _ptr(tiles), _ptr(items),
                                            items.shape[0], _ptr(k_cache), _ptr(v_cache),
                                            k_cache.shape[2], k_cache.shape[0], _stream()),
          "slx_attention_prefill")
    return out


@_op("silu_mul", 1)
def silu_mul_blocked(out, gu, ffn: int):
    check(_lib.load().slx_silu_mul_blocked(_dt(out), _ptr(out), _ld(out), _ptr(gu), _ld(gu),
                                           gu.shape[0], ffn, _stream()), "slx_silu_mul_blocked")
    return out


@_op("argmax", 1)
def argmax(out, logits):
    check(_lib.load().slx_argmax(_dt(logits), _ptr(out), _ptr(logits), _ld(logits),
                                 logits.shape[0], logits.shape[1], _stream()), "slx_argmax")
    return out
