"""CPU: the C-ABI library loads, exports every symbol include/slora_b200.h declares, and
rejects bad arguments with status codes before touching the device."""

import ctypes
import os
import re

import pytest

from paper_2505_14468_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "slora_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SLX_API\s+[\w\s\*]+?\b(slx_\w+)\s*\(", text)))


def test_header_declares_symbols():
    syms = header_symbols()
    assert len(syms) >= 25
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.slx_abi_version() == _lib.ABI_VERSION


def test_status_strings():
    lib = _lib.load()
    for st in range(0, -7, -1):
        assert lib.slx_status_string(st).decode() != "unknown status"
    with pytest.raises(ValueError):
        _lib.check(_lib.SLX_ERR_INVALID, "x")
    with pytest.raises(_lib.SlxError):
        _lib.check(_lib.SLX_ERR_CUDA, "x")


def test_argument_validation_without_device():
    lib = _lib.load()
    null = None
    # null operands / bad shapes are rejected before any CUDA call
    assert lib.slx_gemm_bf16(null, 64, null, null, 64, 0, null, 0, 1, 128, 64, 0, 0, 0, null, 0, null, 0, null) == -1
    assert lib.slx_pack_weight(null, null, 128, 64, 64, null) == -1
    assert lib.slx_packed_weight_elems(130, 70) == 256 * 128
    assert lib.slx_rmsnorm(0, null, 8, null, 8, null, 1, 7, 1e-5, null) == -1
    assert lib.slx_lora_apply(0, null, 8, null, 8, 1, 8, null, null, 1, 16, 1, None, null, 0, null) == -1
    assert lib.slx_attention(0, null, 128, null, 384, 1, 1, 1, 128, null, null, null, null, 8, null) == -1
    assert lib.slx_lora_workspace_bytes(64, 32, 16, 3) > 0
    assert lib.slx_gemm_workspace_bytes(0, 128, 64, 0) == 0
    assert lib.slx_gemm_workspace_bytes(64, 4096, 4096, 1) > 64 * 1024
    # misaligned pointer
    buf = (ctypes.c_char * 64)()
    addr = ctypes.addressof(buf) | 1
    assert lib.slx_embedding(0, addr, addr, addr, 1, 8, 10, null) == -2


def test_gathered_lora_argument_validation_without_device():
    """slx_lora_expand / slx_lora_shrink reject what their bulk copies cannot move (v rows not
    16-byte aligned: ldv, v_col_off or v_slot_stride not multiples of 4; misaligned v) before any
    CUDA call."""
    LoraTarget = _lib.LoraTarget
    lib = _lib.load()
    buf = (ctypes.c_char * 4096)()
    base = (ctypes.addressof(buf) + 255) // 256 * 256
    tg = (LoraTarget * 1)()
    tg[0] = LoraTarget(base, base, 64, 0, 64, 64)
    offs = (ctypes.c_int * 1)(0)
    ws, wsb = base, 2048
    # ldv not a multiple of 4
    assert lib.slx_lora_expand(0, base, 64, base, 66, 4, base, base, 2, 16, 1, tg, offs, 0,
                               ws, wsb, None) == -1
    # v_slot_stride not a multiple of 4
    assert lib.slx_lora_expand(0, base, 64, base, 64, 4, base, base, 2, 16, 1, tg, offs, 18,
                               ws, wsb, None) == -1
    # v_col_off not a multiple of 4
    offs2 = (ctypes.c_int * 1)(2)
    assert lib.slx_lora_expand(0, base, 64, base, 64, 4, base, base, 2, 16, 1, tg, offs2, 0,
                               ws, wsb, None) == -1
    # misaligned v
    assert lib.slx_lora_expand(0, base, 64, base + 4, 64, 4, base, base, 2, 16, 1, tg, offs, 0,
                               ws, wsb, None) == -2
    # shrink: max_rank beyond the 64-row limit, misaligned x
    assert lib.slx_lora_shrink(0, base, 64, base, 64, 4, 64, base, 2, 128, 1, tg, offs, ws, wsb,
                               None) == -1
    assert lib.slx_lora_shrink(0, base, 64, base + 2, 64, 4, 64, base, 2, 16, 1, tg, offs, ws, wsb,
                               None) == -2
