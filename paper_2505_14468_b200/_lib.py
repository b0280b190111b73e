"""ctypes binding of libslora_b200.so (the C ABI in include/slora_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` / ``make -C
paper_2505_14468_b200/csrc``.  There is no fallback: if the shared object is
missing every op raises, so a GPU run can never silently take another path.
"""

from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libslora_b200.so")

ABI_VERSION = 2
SLX_OK = 0
SLX_ERR_INVALID = -1
SLX_ERR_ALIGN = -2
SLX_ERR_UNSUPPORTED = -3
SLX_ERR_WORKSPACE = -4
SLX_ERR_CUDA = -5
SLX_ERR_NCCL = -6

DT_BF16 = 0
DT_F32 = 1
EPI_NONE = 0
EPI_RESIDUAL = 1
EPI_SILU_MUL = 2
W_ROWMAJOR = 0
W_TILED = 1
LORA_MAX_TARGETS = 4

_p = ctypes.c_void_p
_i = ctypes.c_int
_f = ctypes.c_float
_sz = ctypes.c_size_t


class LoraTarget(ctypes.Structure):
    _fields_ = [("a_ptrs", _p), ("b_ptrs", _p), ("d_out", _i), ("y_col_offset", _i),
                ("y_col_block", _i), ("y_col_stride", _i)]


class LoraDelta(ctypes.Structure):
    """slx_lora_delta: fused decode expand in a consumer kernel."""
    _fields_ = [("v", _p), ("ldv", _i), ("tok_slot", _p), ("slot_rank", _p), ("slot_scale", _p),
                ("max_rank", _i), ("n_targets", _i), ("v_slot_stride", _i), ("b_ptrs", _p * 4),
                ("v_col_off", _i * 4),
                ("y_col_off", _i * 4), ("d_out", _i * 4)]


class SplitKIn(ctypes.Structure):
    """slx_splitk_in: split-K pieces of a projection for the consuming kernel."""
    _fields_ = [("part", _p), ("splits", _i), ("bm", _i), ("n_main", _i)]


class GemmTuning(ctypes.Structure):
    """slx_gemm_tuning: explicit tiling for tests / tools (all zero = the planner's choice)."""
    _fields_ = [("tile_kernel", _i), ("ctas_per_sm", _i), ("splits", _i), ("bn", _i),
                ("gsplit", _i), ("sk_ctas", _i), ("sk_min_units", _i), ("sk_no_cluster", _i)]


class RopeKV(ctypes.Structure):
    """slx_rope_kv: RoPE + KV append fused into the q/k/v projection's epilogue."""
    _fields_ = [("tok_pos", _p), ("tok_seq", _p), ("cos_tab", _p), ("sin_tab", _p), ("max_pos", _i),
                ("k_cache", _p), ("v_cache", _p), ("max_ctx", _i), ("heads", _i), ("kv_heads", _i),
                ("head_dim", _i)]


class L2Prefetch(ctypes.Structure):
    """slx_l2_prefetch: the next kernel's first bytes (two regions)."""
    _fields_ = [("ptr", _p * 2), ("bytes", _sz * 2)]


# name -> (restype, argtypes): every symbol declared in include/slora_b200.h
SIGNATURES = {
    "slx_status_string": (ctypes.c_char_p, [_i]),
    "slx_abi_version": (_i, []),
    "slx_device_sm_count": (_i, [ctypes.POINTER(_i)]),
    "slx_gemm_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "slx_gemm_bf16": (_i, [_p, _i, _p, _p, _i, _i, _p, _i, _i, _i, _i, _i, _i, _i, _p, _i, _p, _sz,
                           _p]),
    "slx_debug_gemm_trace": (_i, [_p]),
    "slx_gemm_splitk_bytes": (_sz, [_i, _i, _i]),
    "slx_gemm_bf16_splitk": (_i, [_p, _i, _p, _i, _i, _i, _i, _p, _sz, ctypes.POINTER(L2Prefetch), _p]),
    "slx_gemm_bf16_ex": (_i, [_p, _i, _p, _p, _i, _i, _p, _i, _i, _i, _i, _i, _i, _i, _p, _i, _p,
                              _sz, ctypes.POINTER(L2Prefetch), ctypes.POINTER(GemmTuning), _p]),
    "slx_pack_weight_rows": (_i, [_p, _p, _i, _i, _i, _i, _p]),
    "slx_gemm_group_tile_bytes": (_sz, []),
    "slx_gemm_bf16_lorafold": (_i, [_p, _i, _p, _i, _p, _i, _i, _p, _i, _i, _i, _i, _i, _p, _i, _p, _i,
                                    _i, _p, _i, _p, _p, _p, ctypes.POINTER(RopeKV), _p]),
    "slx_gemm_grouped_bf16": (_i, [_p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _i, _i, _p, _i,
                                   _i, _i, _p, _i, _p]),
    "slx_lora_expand": (_i, [_i, _p, _i, _p, _i, _i, _p, _p, _i, _i, _i,
                             ctypes.POINTER(LoraTarget), ctypes.POINTER(_i), _i, _p, _sz, _p]),
    "slx_lora_shrink": (_i, [_i, _p, _i, _p, _i, _i, _i, _p, _i, _i, _i,
                             ctypes.POINTER(LoraTarget), ctypes.POINTER(_i), _p, _sz, _p]),
    "slx_packed_weight_elems": (_sz, [_i, _i]),
    "slx_pack_weight": (_i, [_p, _p, _i, _i, _i, _p]),
    "slx_gemm_f32": (_i, [_p, _i, _p, _p, _i, _p, _i, _i, _i, _i, _i, _p]),
    "slx_lora_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "slx_lora_plan_tokens": (_i, [_p, _i, _i, _p, _sz, _p]),
    "slx_lora_plan_segments": (_i, [_p, _p, _i, _i, _i, _p, _sz, _p]),
    "slx_lora_apply": (_i, [_i, _p, _i, _p, _i, _i, _i, _p, _p, _i, _i, _i,
                            ctypes.POINTER(LoraTarget), _p, _sz, _p]),
    "slx_lora_bgmv": (_i, [_i, _p, _i, _p, _i, _p, _i, _i, _p, _p, _i, _i, _i,
                           ctypes.POINTER(LoraTarget), _p, _sz, _p]),
    "slx_lora_sgmv": (_i, [_i, _p, _i, _p, _i, _p, _p, _i, _i, _i, _p, _p, _i, _i, _i,
                           ctypes.POINTER(LoraTarget), _p, _sz, _p]),
    "slx_embedding": (_i, [_i, _p, _p, _p, _i, _i, _i, _p]),
    "slx_rmsnorm": (_i, [_i, _p, _i, _p, _i, _p, _i, _i, _f, _p]),
    "slx_rmsnorm_lora": (_i, [_i, _p, _i, _p, _i, _p, _i, _i, _f, ctypes.POINTER(LoraDelta), _p]),
    "slx_rmsnorm_fused": (_i, [_i, _p, _i, _p, _i, _p, _i, _i, _f, ctypes.POINTER(SplitKIn),
                               ctypes.POINTER(LoraDelta), ctypes.POINTER(L2Prefetch), _p]),
    "slx_rope_kv_write": (_i, [_i, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _i, _p, _p, _i, _p]),
    "slx_attention": (_i, [_i, _p, _i, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _i, _p]),
    "slx_rope_attention_decode": (_i, [_i, _p, _i, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _i,
                                       _p, _p, _i, _i, ctypes.POINTER(LoraDelta),
                                       ctypes.POINTER(L2Prefetch), _p]),
    "slx_flash_prefill_tile_queries": (_i, []),
    "slx_flash_prefill_tile_bytes": (_sz, []),
    "slx_flash_prefill_item_bytes": (_sz, []),
    "slx_attention_prefill": (_i, [_p, _i, _p, _i, _i, _i, _i, _i, _p, _p, _i, _p, _p, _i, _i, _p]),
    "slx_silu_mul_blocked": (_i, [_i, _p, _i, _p, _i, _i, _i, _p]),
    "slx_argmax": (_i, [_i, _p, _p, _i, _i, _i, _p]),
    "slx_host_register": (_i, [_p, _sz]),
    "slx_host_unregister": (_i, [_p]),
    "slx_preload_h2d": (_i, [_p, _p, _sz, _sz, _p, _p]),
    "slx_offload_d2h": (_i, [_p, _p, _sz, _sz, _p, _p]),
    "slx_nccl_unique_id_bytes": (_i, []),
    "slx_nccl_get_unique_id": (_i, [_p]),
    "slx_nccl_comm_init": (_i, [ctypes.POINTER(_p), _i, _p, _i]),
    "slx_nccl_comm_destroy": (_i, [_p]),
    "slx_bcast": (_i, [_p, _sz, _i, _p, _p]),
    "slx_preload_bcast": (_i, [_p, _p, _sz, _sz, _i, _p, _p, _p]),
}

_LIB = None


class SlxError(RuntimeError):
    """A CUDA/NCCL failure reported by libslora_b200."""


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built — no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_2505_14468_b200/csrc)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.slx_abi_version() != ABI_VERSION:
            raise ImportError("libslora_b200 ABI version mismatch")
        _LIB = lib
    return _LIB


def check(status: int, what: str) -> None:
    if status == SLX_OK:
        return
    msg = f"{what}: {load().slx_status_string(status).decode()} (status {status})"
    if status in (SLX_ERR_INVALID, SLX_ERR_ALIGN, SLX_ERR_UNSUPPORTED, SLX_ERR_WORKSPACE):
        raise ValueError(msg)
    raise SlxError(msg)
