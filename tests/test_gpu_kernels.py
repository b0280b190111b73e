"""GPU: each kernel against the oracle (LoRA, ops) or a plain torch fp32 reference (GEMM)."""

import numpy as np
import pytest
import torch

from oracle import llama_lora as orc
from paper_2505_14468_b200 import ops
from paper_2505_14468_b200._lib import EPI_NONE, EPI_RESIDUAL, EPI_SILU_MUL

pytestmark = pytest.mark.gpu
DEV = "cuda"


def bf(x):
    return x.to(torch.bfloat16)


# ------------------------------------------------------------------ K1 GEMM
GEMM_SHAPES = [
    (1, 128, 64), (7, 256, 128), (16, 4096, 4096), (64, 12288, 4096), (64, 4096, 11008),
    (100, 384, 688), (128, 1024, 512), (129, 512, 256), (300, 768, 320), (1024, 4096, 4096),
    (2048, 256, 4096), (64, 32000, 4096),
]


@pytest.mark.parametrize("tiled", [False, True])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_matches_torch_fp32(M, N, K, tiled):
    g = torch.Generator(device=DEV).manual_seed(M * 7 + N + K)
    a = bf(torch.randn(M, K, device=DEV, generator=g))
    w = bf(torch.randn(N, K, device=DEV, generator=g) * 0.05)
    ref = a.float() @ w.float().T
    wk = ops.pack_weight(w) if tiled else w
    out32 = ops.gemm(a, wk, out_dtype=torch.float32)
    torch.cuda.synchronize()
    torch.testing.assert_close(out32, ref, rtol=1e-4, atol=1e-3)   # fp32 out: accumulation order only
    out = ops.gemm(a, wk)
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M", [1, 64, 100])
@pytest.mark.parametrize("bn", [256, 128])
@pytest.mark.parametrize("gsplit", [0, 1])
@pytest.mark.parametrize("ctas,splits", [(1, 1), (2, 8), (1, 3), (1, 6), (2, 2), (1, 5)])
def test_gemm_decode_tilings(M, bn, gsplit, ctas, splits):
    """Every cluster / global split-K tiling of the tile kernel gives the same result (explicit
    slx_gemm_tuning; the stream-K decode kernel is bypassed)."""
    N, K = 3072, 4096
    a = bf(torch.randn(M, K, device=DEV))
    w = bf(torch.randn(N, K, device=DEV) * 0.05)
    ref = a.float() @ w.float().T
    tu = {"tile_kernel": 1, "ctas_per_sm": ctas, "splits": splits, "bn": bn,
          "gsplit": 1 if gsplit else 2}
    out = ops.gemm(a, ops.pack_weight(w), out_dtype=torch.float32, tuning=tu)
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-3)
    # SiLU and residual epilogues through the same split-K reduction
    r = torch.randn(M, N, device=DEV)   # residual has the output dtype
    o2 = ops.gemm(a, ops.pack_weight(w), epilogue=EPI_RESIDUAL, residual=r, out_dtype=torch.float32,
                  tuning=tu)
    torch.testing.assert_close(o2, ref + r, rtol=1e-4, atol=1e-3)
    g_, u_ = ref.view(M, N // 256, 2, 128)[:, :, 0], ref.view(M, N // 256, 2, 128)[:, :, 1]
    tu["bn"] = 256   # SiLU pairs always use 256-wide tiles
    o3 = ops.gemm(a, ops.pack_weight(w), epilogue=EPI_SILU_MUL, out_dtype=torch.float32, tuning=tu)
    torch.testing.assert_close(o3, (g_ * torch.sigmoid(g_) * u_).reshape(M, N // 2), rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("M", [1, 17, 64, 65, 100, 128])
@pytest.mark.parametrize("N,K", [(3072, 4096), (4608, 4096), (1000, 11008), (32000, 1024)])
@pytest.mark.parametrize("ctas,min_units,cluster", [(0, 4, 1), (0, 4, 0), (37, 4, 1), (5, 4, 1),
                                                     (1, 1, 1), (0, 1, 1)])
def test_gemm_stream_k(M, N, K, ctas, min_units, cluster):
    """Stream-K decode GEMM (M <= 128; M = 64 / M = 128 MMAs): every range split (whole tiles, tail/head pieces, up to
    dozens of pieces per tile; uniform splits reduced in DSMEM clusters or through global
    memory) gives the fp32 result; epilogues residual / SiLU / side output."""
    tu = {"sk_no_cluster": 0 if cluster else 1, "sk_ctas": ctas, "sk_min_units": min_units}
    g = torch.Generator(device=DEV).manual_seed(M + N + K + ctas)
    a = bf(torch.randn(M, K, device=DEV, generator=g))
    w = bf(torch.randn(N, K, device=DEV, generator=g) * 0.05)
    ref = a.float() @ w.float().T
    pw = ops.pack_weight(w)
    out = ops.gemm(a, pw, out_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-3)
    again = ops.gemm(a, pw, out_dtype=torch.float32)   # counters re-armed, same split order
    assert torch.equal(out, again)
    r = bf(torch.randn(M, N, device=DEV, generator=g))
    o2 = ops.gemm(a, pw, epilogue=EPI_RESIDUAL, residual=r)
    torch.testing.assert_close(o2.float(), ref + r.float(), rtol=1e-2, atol=2e-2)
    if N % 256 == 0:
        g_, u_ = ref.view(M, N // 256, 2, 128)[:, :, 0], ref.view(M, N // 256, 2, 128)[:, :, 1]
        o3 = ops.gemm(a, pw, epilogue=EPI_SILU_MUL, out_dtype=torch.float32)
        torch.testing.assert_close(o3, (g_ * torch.sigmoid(g_) * u_).reshape(M, N // 2), rtol=1e-3,
                                   atol=1e-3)
    # stacked extra rows -> fp32 side output (decode LoRA shrink), main columns + residual
    if N % 128:
        return
    E = 512
    ext = bf(torch.randn(E, K, device=DEV, generator=g) * 0.05)
    pw2 = ops.pack_weight(w, extra_rows=E)
    ops.pack_rows(pw2, ext, E, N)
    x = r.clone()
    side = torch.empty(M, E, device=DEV)
    ops.gemm(a, pw2, x, epilogue=EPI_RESIDUAL, residual=x, side=side)
    torch.testing.assert_close(x.float(), ref + r.float(), rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(side, a.float() @ ext.float().T, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M", [3, 64, 200])
def test_gemm_residual_inplace(M):
    N, K = 512, 256
    g = torch.Generator(device=DEV).manual_seed(M)
    a = bf(torch.randn(M, K, device=DEV, generator=g))
    w = bf(torch.randn(N, K, device=DEV, generator=g) * 0.05)
    x = bf(torch.randn(M, N, device=DEV, generator=g))
    ref = a.float() @ w.float().T + x.float()
    ops.gemm(a, ops.pack_weight(w), x, epilogue=EPI_RESIDUAL, residual=x)
    torch.testing.assert_close(x.float(), ref, rtol=1e-2, atol=2e-2)


@pytest.mark.parametrize("M", [1, 64, 300])
def test_gemm_silu_mul_blocked(M):
    F, K = 384, 256
    g = torch.Generator(device=DEV).manual_seed(M + 1)
    a = bf(torch.randn(M, K, device=DEV, generator=g))
    gate = bf(torch.randn(F, K, device=DEV, generator=g) * 0.05)
    up = bf(torch.randn(F, K, device=DEV, generator=g) * 0.05)
    w = torch.stack([gate.view(F // 128, 128, K), up.view(F // 128, 128, K)], 1).reshape(2 * F, K).contiguous()
    gr, ur = a.float() @ gate.float().T, a.float() @ up.float().T
    ref = gr * torch.sigmoid(gr) * ur
    out = ops.gemm(a, w, epilogue=EPI_SILU_MUL, out_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=1e-3)
    out = ops.gemm(a, ops.pack_weight(w), epilogue=EPI_SILU_MUL, out_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=1e-3)


def test_gemm_deterministic_split_k():
    a = bf(torch.randn(64, 4096, device=DEV))
    w = bf(torch.randn(4096, 4096, device=DEV) * 0.02)
    o1 = ops.gemm(a, w, out_dtype=torch.float32)
    o2 = ops.gemm(a, w, out_dtype=torch.float32)
    assert torch.equal(o1, o2)


def test_gemm_f32_parity():
    a = torch.randn(37, 200, device=DEV)
    w = bf(torch.randn(72, 200, device=DEV))
    r = torch.randn(37, 72, device=DEV)
    out = ops.gemm_f32(a, w, residual=r)
    ref = (a.double() @ w.double().T + r.double()).float()
    torch.testing.assert_close(out, ref, rtol=1e-5, atol=1e-4)


# ------------------------------------------------------------------ K2/K3 LoRA
def _adapters(n_slots, ranks, d_in, d_outs, seed):
    rng = np.random.default_rng(seed)
    pools = []
    for d_out in d_outs:
        A = [rng.standard_normal((r, d_in)).astype(np.float32) / np.sqrt(d_in) for r in ranks]
        B = [rng.standard_normal((d_out, r)).astype(np.float32) * 0.05 for r in ranks]
        A = [orc_round(a) for a in A]
        B = [orc_round(b) for b in B]
        pools.append((A, B))
    return pools


def orc_round(x):
    from paper_2505_14468_b200.config import round_to_bf16
    return round_to_bf16(x)


def _targets(pools, d_outs):
    keep, specs = [], []
    off = 0
    for (A, B), d_out in zip(pools, d_outs):
        At = [torch.from_numpy(a).to(DEV, torch.bfloat16) for a in A]
        Bt = [torch.from_numpy(b).to(DEV, torch.bfloat16) for b in B]
        keep += At + Bt
        ap = torch.tensor([t.data_ptr() for t in At], dtype=torch.int64, device=DEV)
        bp = torch.tensor([t.data_ptr() for t in Bt], dtype=torch.int64, device=DEV)
        keep += [ap, bp]
        specs.append((ap, bp, d_out, off, d_out, d_out))
        off += d_out
    return ops.make_targets(specs), keep


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("T,n_slots,d_in,d_outs,ranks", [
    (64, 32, 4096, (4096, 4096, 4096), [16] * 32),          # config-2 decode shape (q,k,v)
    (1, 4, 256, (256,), [8] * 4),
    (37, 6, 512, (384, 128), [8, 16, 64, 8, 16, 64]),       # mixed ranks
])
def test_bgmv_matches_oracle(dtype, T, n_slots, d_in, d_outs, ranks):
    rng = np.random.default_rng(T + n_slots)
    pools = _adapters(n_slots, ranks, d_in, d_outs, seed=n_slots)
    tok_slot = rng.integers(-1, n_slots, size=T).astype(np.int32)
    x = orc_round(rng.standard_normal((T, d_in)).astype(np.float32))
    y0 = orc_round(rng.standard_normal((T, sum(d_outs))).astype(np.float32))
    scales = [2.0 + 0.25 * s for s in range(n_slots)]
    ref = y0.copy()
    off = 0
    for (A, B), d_out in zip(pools, d_outs):
        ref[:, off:off + d_out] = orc.bgmv(y0[:, off:off + d_out], x, A, B, scales, tok_slot)
        off += d_out
    targets, keep = _targets(pools, d_outs)
    xd = torch.from_numpy(x).to(DEV, dtype)
    yd = torch.from_numpy(y0).to(DEV, dtype)
    rank = torch.tensor(ranks, dtype=torch.int32, device=DEV)
    scale = torch.tensor(scales, dtype=torch.float32, device=DEV)
    wsb = torch.zeros(ops.lora_workspace_bytes(T, n_slots, 64, len(d_outs)), dtype=torch.uint8, device=DEV)
    ops.lora_bgmv(yd, xd, torch.from_numpy(tok_slot).to(DEV), rank, scale, 64, targets, wsb)
    got = yd.float().cpu().numpy()
    if dtype == torch.float32:
        np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5)
    else:
        np.testing.assert_allclose(got, ref, rtol=2e-2, atol=3e-2)
        # untouched rows (slot -1) stay bit-identical
        none = tok_slot < 0
        assert np.array_equal(got[none], y0[none])


@pytest.mark.parametrize("seg_lens", [[5, 0, 17, 1, 33], [2048, 2048], [1]])
def test_sgmv_matches_oracle(seg_lens):
    rng = np.random.default_rng(len(seg_lens))
    n_slots, d_in, d_out = 5, 640, 512
    ranks = [8, 16, 64, 16, 8]
    pools = _adapters(n_slots, ranks, d_in, (d_out,), seed=3)
    T = sum(seg_lens)
    seg_indptr = np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int32)
    seg_slot = np.asarray([(i * 2) % n_slots for i in range(len(seg_lens))], np.int32)
    x = orc_round(rng.standard_normal((T, d_in)).astype(np.float32))
    y0 = rng.standard_normal((T, d_out)).astype(np.float32)
    scales = [1.0, 2.0, 0.5, 1.5, 3.0]
    A, B = pools[0]
    ref = orc.sgmv(y0, x, A, B, scales, seg_indptr, seg_slot)
    targets, keep = _targets(pools, (d_out,))
    yd = torch.from_numpy(y0).to(DEV)
    wsb = torch.zeros(ops.lora_workspace_bytes(T, n_slots, 64, 1), dtype=torch.uint8, device=DEV)
    ops.lora_sgmv(yd, torch.from_numpy(x).to(DEV), torch.from_numpy(seg_indptr).to(DEV),
                  torch.from_numpy(seg_slot).to(DEV), torch.tensor(ranks, dtype=torch.int32, device=DEV),
                  torch.tensor(scales, device=DEV), 64, targets, wsb)
    np.testing.assert_allclose(yd.cpu().numpy(), ref, rtol=1e-4, atol=1e-4)


# ------------------------------------------------------------------ K4 ops
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rmsnorm_embedding_argmax(dtype):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((9, 4096)).astype(np.float32)
    w = orc_round(1 + 0.1 * rng.standard_normal(4096).astype(np.float32))
    out = torch.empty(9, 4096, dtype=dtype, device=DEV)
    xd = torch.from_numpy(x).to(DEV, dtype)
    ops.rmsnorm(out, xd, torch.from_numpy(w).to(DEV, torch.bfloat16), 1e-5)
    ref = orc.rmsnorm(xd.float().cpu().numpy(), w, 1e-5)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    np.testing.assert_allclose(out.float().cpu().numpy(), ref, rtol=tol, atol=tol)
    table = orc_round(rng.standard_normal((100, 256)).astype(np.float32))
    toks = np.array([3, 99, 0, 3], np.int32)
    e = torch.empty(4, 256, dtype=dtype, device=DEV)
    ops.embedding(e, torch.from_numpy(table).to(DEV, torch.bfloat16), torch.from_numpy(toks).to(DEV))
    assert np.array_equal(e.float().cpu().numpy(), table[toks])
    lg = rng.standard_normal((6, 32000)).astype(np.float32)
    lg[2, 7] = lg[2, 9] = 100.0  # tie -> lowest index (different 16-byte chunks)
    lg[3, 5] = lg[3, 6] = 100.0  # tie inside one 16-byte chunk
    lg[4, 31999] = lg[4, 4 * 512 + 1] = 100.0   # tie across threads of the vectorised scan
    lg[5, :] = -3.0              # all equal -> index 0
    am = torch.empty(6, dtype=torch.int32, device=DEV)
    ops.argmax(am, torch.from_numpy(lg).to(DEV))
    assert am.cpu().numpy().tolist() == np.argmax(lg, -1).tolist()
    am2 = torch.empty(6, dtype=torch.int32, device=DEV)   # odd width: the scalar scan
    ops.argmax(am2, torch.from_numpy(np.ascontiguousarray(lg[:, :31999])).to(DEV))
    assert am2.cpu().numpy().tolist() == np.argmax(lg[:, :31999], -1).tolist()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("H,Hkv,D", [(4, 4, 64), (8, 2, 128)])
def test_rope_kv_attention_match_oracle(dtype, H, Hkv, D):
    rng = np.random.default_rng(H + D)
    lens = [1, 13, 70, 200]       # one prefill chunk per sequence, ragged
    T = sum(lens)
    max_ctx = 256
    qkv = rng.standard_normal((T, (H + 2 * Hkv) * D)).astype(np.float32)
    pos = np.concatenate([np.arange(L) for L in lens]).astype(np.int32)
    seq = np.concatenate([[s] * L for s, L in enumerate(lens)]).astype(np.int32)
    cos, sin = orc.rope_table(max_ctx, D, 10000.0)
    kc = torch.zeros(len(lens), Hkv, max_ctx, D, dtype=dtype, device=DEV)
    vc = torch.zeros_like(kc)
    qd = torch.from_numpy(qkv).to(DEV, dtype)
    qkv_r = qd.float().cpu().numpy()
    ops.rope_kv_write(qd, H, Hkv, D, torch.from_numpy(pos).to(DEV), torch.from_numpy(seq).to(DEV),
                      torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV), kc, vc)
    out = torch.empty(T, H * D, dtype=dtype, device=DEV)
    ops.attention(out, qd, H, Hkv, D, torch.from_numpy(pos).to(DEV), torch.from_numpy(seq).to(DEV), kc, vc)
    q = orc.apply_rope(qkv_r[:, :H * D].reshape(T, H, D), pos, cos, sin)
    k = orc.apply_rope(qkv_r[:, H * D:(H + Hkv) * D].reshape(T, Hkv, D), pos, cos, sin)
    v = qkv_r[:, (H + Hkv) * D:].reshape(T, Hkv, D)
    ref = np.empty((T, H, D), np.float32)
    o = 0
    for L in lens:
        ref[o:o + L] = orc.attention(q[o:o + L], k[o:o + L], v[o:o + L], np.arange(L))
        o += L
    tol = 2e-5 if dtype == torch.float32 else 3e-2
    np.testing.assert_allclose(out.float().cpu().numpy(), ref.reshape(T, -1), rtol=tol, atol=tol)
    np.testing.assert_allclose(kc[1, :, :13].float().cpu().numpy().transpose(1, 0, 2), k[1:14], rtol=tol, atol=tol)


@pytest.mark.parametrize("dtype", [torch.bfloat16])
@pytest.mark.parametrize("H,Hkv,D", [(4, 4, 64), (8, 2, 128)])
def test_rope_kv_vectorised_equals_scalar(dtype, H, Hkv, D):
    """The 16-byte vectorised bf16 RoPE + KV write (aligned rows) == the scalar kernel
    (unaligned row stride), bit for bit: rotated q/k in place and the appended k/v."""
    g = torch.Generator(device=DEV).manual_seed(D)
    T, W = 37, (H + 2 * Hkv) * D
    base = torch.randn(T, W, generator=g, device=DEV).to(dtype)
    pos = torch.arange(T, dtype=torch.int32, device=DEV) // 5 + 3   # unique (seq, pos) rows
    seq = torch.arange(T, dtype=torch.int32, device=DEV) % 5
    cos, sin = (torch.from_numpy(t).to(DEV) for t in orc.rope_table(64, D, 10000.0))
    res = []
    for ld in (W, W + 1):   # ld % 8 != 0 forces the scalar kernel
        buf = torch.zeros(T, ld, dtype=dtype, device=DEV)
        buf[:, :W] = base
        kc = torch.zeros(5, Hkv, 64, D, dtype=dtype, device=DEV)
        vc = torch.zeros_like(kc)
        ops.rope_kv_write(buf[:, :W], H, Hkv, D, pos, seq, cos, sin, kc, vc)
        res.append((buf[:, :W].clone(), kc, vc))
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("H,Hkv,D", [(4, 4, 64), (32, 32, 128), (8, 2, 128)])
@pytest.mark.parametrize("ctx", [0, 5, 128, 300])
def test_rope_attention_decode_fused(dtype, H, Hkv, D, ctx):
    """Fused decode kernel == rope_kv_write + attention (and the oracle), incl. the KV append."""
    rng = np.random.default_rng(ctx + D)
    B, max_ctx = 3, 320
    cos, sin = orc.rope_table(max_ctx, D, 10000.0)
    cos_d, sin_d = torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV)
    kc = torch.from_numpy(rng.standard_normal((B, Hkv, max_ctx, D)).astype(np.float32)).to(DEV, dtype)
    vc = torch.from_numpy(rng.standard_normal((B, Hkv, max_ctx, D)).astype(np.float32)).to(DEV, dtype)
    qkv = torch.from_numpy(rng.standard_normal((B, (H + 2 * Hkv) * D)).astype(np.float32)).to(DEV, dtype)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=DEV)
    seq = torch.arange(B, dtype=torch.int32, device=DEV)
    kc2, vc2, qkv2 = kc.clone(), vc.clone(), qkv.clone()
    out_f = torch.empty(B, H * D, dtype=dtype, device=DEV)
    ops.rope_attention_decode(out_f, qkv, H, Hkv, D, pos, seq, cos_d, sin_d, kc, vc)
    out_u = torch.empty(B, H * D, dtype=dtype, device=DEV)
    ops.rope_kv_write(qkv2, H, Hkv, D, pos, seq, cos_d, sin_d, kc2, vc2)
    ops.attention(out_u, qkv2, H, Hkv, D, pos, seq, kc2, vc2)
    tol = 2e-5 if dtype == torch.float32 else 2e-2
    torch.testing.assert_close(out_f.float(), out_u.float(), rtol=tol, atol=tol)
    assert torch.equal(kc[:, :, :ctx + 1], kc2[:, :, :ctx + 1])   # identical KV append
    assert torch.equal(vc[:, :, :ctx + 1], vc2[:, :, :ctx + 1])
    # oracle: rotate q/k in fp32 from the (dtype-rounded) inputs
    q_in = qkv.float().cpu().numpy() if dtype == torch.float32 else qkv2.float().cpu().numpy()
    kk = kc2[:, :, :ctx + 1].float().cpu().numpy()
    vv = vc2[:, :, :ctx + 1].float().cpu().numpy()
    for b in range(B):
        q = q_in[b, :H * D].reshape(1, H, D)
        if dtype == torch.float32:
            q = orc.apply_rope(q, np.array([ctx]), cos, sin)
        ref = orc.attention(q, kk[b].transpose(1, 0, 2), vv[b].transpose(1, 0, 2), np.array([ctx]))
        np.testing.assert_allclose(out_f[b].float().cpu().numpy(), ref.reshape(-1), rtol=tol * 5, atol=tol * 5)


def _decode_attention_oracle(qkv, kc, vc, pos, seq, slot, ranks, scales, v_all, Bs, H, D, cos, sin,
                             n_slots, rank):
    """fp32 numpy restatement of the fused decode step for every token: q/k/v rows + their LoRA
    delta (rounded to bf16 like the kernel), rotate-half RoPE at pos (oracle/llama_lora.py),
    append, attention over the sequence's positions 0..pos (oracle attention)."""
    qkv = qkv.float().cpu().numpy()
    kcn, vcn = kc.float().cpu().numpy(), vc.float().cpu().numpy()
    v_all = v_all.cpu().numpy()
    Bn = [b.float().cpu().numpy() for b in Bs]
    slot, ranks, scales = slot.cpu().numpy(), ranks.cpu().numpy(), scales.cpu().numpy()
    pos, seq = pos.cpu().numpy(), seq.cpu().numpy()
    bfr = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().float().numpy()  # noqa: E731
    outs, news = [], []
    for b in range(qkv.shape[0]):
        row = qkv[b].copy()
        s_ = int(slot[b])
        if s_ >= 0:
            r = int(ranks[s_])
            for i in range(3):
                v = v_all[b, i * n_slots * rank + s_ * rank: i * n_slots * rank + s_ * rank + r] * scales[s_]
                row[i * H * D:(i + 1) * H * D] += Bn[i][s_][:, :r] @ v
            row = bfr(row)
        q = row[:H * D].reshape(1, H, D)
        k = row[H * D:2 * H * D].reshape(1, H, D)
        vv = row[2 * H * D:].reshape(1, H, D)
        p_ = np.array([pos[b]])
        q = bfr(orc.apply_rope(q, p_, cos, sin))
        k = bfr(orc.apply_rope(k, p_, cos, sin))
        ks = np.concatenate([kcn[seq[b], :, :pos[b]].transpose(1, 0, 2), k], 0)
        vs = np.concatenate([vcn[seq[b], :, :pos[b]].transpose(1, 0, 2), vv], 0)
        outs.append(orc.attention(q, ks, vs, p_).reshape(-1))
        news.append((k[0], vv[0]))
    return np.stack(outs), news


@pytest.mark.parametrize("ctx", [0, 1, 127, 128, 129, 300, 512, 1000])
@pytest.mark.parametrize("B,H,D,rank", [(24, 32, 128, 16), (5, 4, 64, 8), (7, 8, 128, 64),
                                        (64, 32, 128, 16)])
def test_attention_decode_pipe_lora(B, H, D, rank, ctx):
    """Persistent TMA-pipelined tensor-core decode attention (several items per CTA,
    multi-block contexts) with the fused q/k/v LoRA delta == the per-(token, head) kernel and
    == the oracle (contexts up to 1000); ranks staged (<= 16) and not staged (64); tokens
    without an adapter; identical KV append.  Long contexts with 14 items per CTA exercise the
    shared KV ring's guard against a consumer group waiting two laps ahead of the producer."""
    rng = np.random.default_rng(ctx + B + rank)
    max_ctx, n_slots = max(320, ctx + 8), 3
    cos, sin = orc.rope_table(max_ctx, D, 10000.0)
    cos_d, sin_d = torch.from_numpy(cos).to(DEV), torch.from_numpy(sin).to(DEV)
    kc = bf(torch.from_numpy(rng.standard_normal((B, H, max_ctx, D)).astype(np.float32)).to(DEV))
    vc = bf(torch.from_numpy(rng.standard_normal((B, H, max_ctx, D)).astype(np.float32)).to(DEV))
    qkv = bf(torch.from_numpy(rng.standard_normal((B, 3 * H * D)).astype(np.float32)).to(DEV))
    pos = torch.full((B,), ctx, dtype=torch.int32, device=DEV)
    seq = torch.from_numpy(rng.permutation(B).astype(np.int32)).to(DEV)
    slot = torch.from_numpy(rng.integers(-1, n_slots, size=B).astype(np.int32)).to(DEV)
    ranks = torch.full((n_slots,), rank, dtype=torch.int32, device=DEV)
    scales = torch.tensor([0.5, 2.0, 1.0], device=DEV)
    v_all = torch.randn(B, 3 * n_slots * rank, device=DEV)
    Bs = [bf(torch.randn(n_slots, H * D, rank, device=DEV) * 0.1) for _ in range(3)]
    tabs = [torch.tensor([b[s].data_ptr() for s in range(n_slots)], dtype=torch.int64, device=DEV)
            for b in Bs]
    delta = ops.make_delta(v_all, slot, ranks, scales, rank,
                           [(tabs[i], i * n_slots * rank, i * H * D, H * D) for i in range(3)])
    out = {}
    caches = {}
    for pipe in (True, False):   # pool_seqs = 0: the one-CTA-per-(token, head) kernel
        k2, v2 = kc.clone(), vc.clone()
        o = torch.empty(B, H * D, dtype=torch.bfloat16, device=DEV)
        ops.rope_attention_decode(o, qkv, H, H, D, pos, seq, cos_d, sin_d, k2, v2, lora=delta,
                                  pool_seqs=None if pipe else 0)
        out[pipe], caches[pipe] = o, (k2, v2)
    torch.cuda.synchronize()
    torch.testing.assert_close(out[True].float(), out[False].float(), rtol=2e-2, atol=2e-2)
    assert torch.equal(caches[True][0], caches[False][0])   # appended k (LoRA + RoPE) identical
    assert torch.equal(caches[True][1], caches[False][1])
    if ctx in (0, 300, 512, 1000) or rank == 64:
        ref, new = _decode_attention_oracle(qkv, kc, vc, pos, seq, slot, ranks, scales, v_all, Bs, H,
                                            D, cos, sin, n_slots, rank)
        np.testing.assert_allclose(out[True].float().cpu().numpy(), ref, rtol=2e-2, atol=2e-2)
        sq = seq.cpu().numpy()
        for b in range(B):
            np.testing.assert_allclose(caches[True][0][sq[b], :, ctx].float().cpu().numpy(), new[b][0],
                                       rtol=1e-2, atol=1e-2)
            np.testing.assert_allclose(caches[True][1][sq[b], :, ctx].float().cpu().numpy(), new[b][1],
                                       rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("d,rank", [(4096, 16), (4096, 64), (5120, 8), (8192, 16)])
def test_rmsnorm_lora_cluster(d, rank):
    """Residual LoRA add + RMSNorm (8-CTA cluster kernel for d % 2048 == 0, one CTA per token
    otherwise) == the fp32 reference; tokens without an adapter untouched."""
    T, n_slots = 37, 4
    g = torch.Generator(device=DEV).manual_seed(d + rank)
    x0 = bf(torch.randn(T, d, device=DEV, generator=g))
    w = bf(torch.rand(d, device=DEV, generator=g) + 0.5)
    slot = torch.randint(-1, n_slots, (T,), device=DEV, generator=g, dtype=torch.int32)
    ranks = torch.full((n_slots,), rank, dtype=torch.int32, device=DEV)
    scales = torch.tensor([0.5, 1.0, 2.0, 4.0], device=DEV)
    v_all = torch.randn(T, n_slots * rank, device=DEV, generator=g)
    Bw = bf(torch.randn(n_slots, d, rank, device=DEV, generator=g) * 0.1)
    tab = torch.tensor([Bw[s].data_ptr() for s in range(n_slots)], dtype=torch.int64, device=DEV)
    delta = ops.make_delta(v_all, slot, ranks, scales, rank, [(tab, 0, 0, d)])
    res = {}
    x = x0.clone()
    h = torch.empty_like(x)
    ops.rmsnorm_lora(h, x, w, 1e-5, delta)
    res["1"] = (x, h)
    torch.cuda.synchronize()
    none = (slot < 0).nonzero().flatten()
    assert torch.equal(res["1"][0][none], x0[none])
    # reference: fp32 delta, bf16 round, fp32 rmsnorm
    sl = slot.clamp(min=0).long()
    dl = torch.einsum("tr,tdr->td", v_all.view(T, n_slots, rank)[torch.arange(T), sl] * scales[sl][:, None],
                      Bw[sl].float())
    xr = torch.where(slot[:, None] >= 0, (x0.float() + dl).bfloat16().float(), x0.float())
    torch.testing.assert_close(res["1"][0].float(), xr, rtol=1e-2, atol=1e-2)
    hr = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    torch.testing.assert_close(res["1"][1].float(), hr, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("M,N,K,splits", [(64, 4608, 4096, 8), (17, 4096, 11008, 8), (1, 512, 256, 3),
                                           (128, 4096, 11008, 8), (100, 4608, 4096, 6)])
def test_gemm_splitk_pieces_and_consumer(M, N, K, splits):
    """Split-K pieces (slx_gemm_bf16_splitk) sum to the fp32 product in the documented layout;
    the fused RMSNorm consumer reproduces residual add + norm."""
    g = torch.Generator(device=DEV).manual_seed(M + N)
    a = bf(torch.randn(M, K, device=DEV, generator=g))
    w = bf(torch.randn(N, K, device=DEV, generator=g) * 0.05)
    ref = a.float() @ w.float().T
    pw = ops.pack_weight(w)
    part = torch.empty(ops.splitk_bytes(M, N, splits) // 4, device=DEV)
    sk = ops.gemm_splitk(a, pw, splits, part)
    bm = (M + 15) // 16 * 16
    pc = part.view(-1, splits, 16, bm, 16)[: (N + 255) // 256]    # [tile][piece][chunk][row][16]
    got = pc.sum(1).permute(2, 0, 1, 3).reshape(bm, -1)[:M, :N]
    torch.testing.assert_close(got, ref, rtol=1e-4, atol=1e-3)
    if N % 2048 == 0 and N <= 8192:
        x0 = bf(torch.randn(M, N, device=DEV, generator=g))
        wn = bf(torch.rand(N, device=DEV, generator=g) + 0.5)
        x, h = x0.clone(), torch.empty_like(x0)
        ops.rmsnorm_fused(h, x, wn, 1e-5, sk)
        xr = (x0.float() + ref).bfloat16().float()
        torch.testing.assert_close(x.float(), xr, rtol=1e-2, atol=2e-2)
        hr = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * wn.float()
        torch.testing.assert_close(h.float(), hr, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("M", [1, 64, 300])
def test_gemm_lora_side_output(M):
    """Stacked extra rows of a packed weight land, in fp32, in the side output; the main
    columns keep the residual epilogue."""
    N, E, K = 512, 384, 4096
    a = bf(torch.randn(M, K, device=DEV))
    w = bf(torch.randn(N, K, device=DEV) * 0.05)
    ext = bf(torch.randn(E, K, device=DEV) * 0.05)
    pw = ops.pack_weight(w, extra_rows=E)
    ops.pack_rows(pw, ext, E, N)
    x = bf(torch.randn(M, N, device=DEV))
    ref_main = a.float() @ w.float().T + x.float()
    side = torch.empty(M, E, device=DEV)
    ops.gemm(a, pw, x, epilogue=EPI_RESIDUAL, residual=x, side=side)
    torch.testing.assert_close(x.float(), ref_main, rtol=1e-2, atol=2e-2)
    torch.testing.assert_close(side, a.float() @ ext.float().T, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("H,Hkv", [(4, 4), (8, 2), (40, 40)])
@pytest.mark.parametrize("segs", [[(0, 1, 0, 0)], [(0, 70, 0, 0), (70, 64, 1, 0), (134, 5, 2, 30)],
                                  [(0, 200, 0, 100), (200, 129, 1, 0)],
                                  [(0, 2048, 0, 0), (2048, 700, 1, 1300), (2748, 130, 2, 0)]])
def test_flash_prefill_matches_oracle(H, Hkv, segs):
    """tcgen05 prefill attention (persistent, paired tiles, lazy rescale) over ragged segments
    with cached prefixes (pos0 > 0), up to 2048 causal keys and more items than SMs."""
    D = 128
    max_ctx = max(320, max(p0 + n for _, n, _, p0 in segs) + 8)
    rng = np.random.default_rng(H + len(segs))
    T = sum(n for _, n, _, _ in segs)
    n_seq = max(s for _, _, s, _ in segs) + 1
    kc = torch.from_numpy(rng.standard_normal((n_seq, Hkv, max_ctx, D)).astype(np.float32)).to(DEV, torch.bfloat16)
    vc = torch.from_numpy(rng.standard_normal((n_seq, Hkv, max_ctx, D)).astype(np.float32)).to(DEV, torch.bfloat16)
    qkv = torch.from_numpy(rng.standard_normal((T, (H + 2 * Hkv) * D)).astype(np.float32)).to(DEV, torch.bfloat16)
    out = torch.empty(T, H * D, dtype=torch.bfloat16, device=DEV)
    plan = ops.prefill_plan(segs, H, DEV)
    ops.attention_prefill(out, qkv, H, Hkv, D, plan, kc, vc)
    # generic attention kernel over the same (already rotated) q and pool
    pos = np.concatenate([np.arange(p0, p0 + n) for _, n, _, p0 in segs]).astype(np.int32)
    seq = np.concatenate([[s] * n for _, n, s, _ in segs]).astype(np.int32)
    ref_k = torch.empty_like(out)
    ops.attention(ref_k, qkv, H, Hkv, D, torch.from_numpy(pos).to(DEV), torch.from_numpy(seq).to(DEV), kc, vc)
    torch.testing.assert_close(out.float(), ref_k.float(), rtol=2e-2, atol=2e-2)
    q = qkv.float().cpu().numpy()[:, :H * D].reshape(T, H, D)
    kk, vv = kc.float().cpu().numpy(), vc.float().cpu().numpy()
    for tok0, n, s_, p0 in segs:
        ref = orc.attention(q[tok0:tok0 + n], kk[s_].transpose(1, 0, 2)[:p0 + n],
                            vv[s_].transpose(1, 0, 2)[:p0 + n], np.arange(p0, p0 + n))
        np.testing.assert_allclose(out[tok0:tok0 + n].float().cpu().numpy(), ref.reshape(n, -1),
                                   rtol=3e-2, atol=3e-2)


@pytest.mark.parametrize("d", [256, 4096, 5120])
def test_rmsnorm_prefill_batch_matches_oracle(d):
    """bf16 RMSNorm of a prefill-sized batch (300 tokens, up to the 13B width) vs the oracle."""
    rng = np.random.default_rng(d)
    T = 300
    x = rng.standard_normal((T, d)).astype(np.float32)
    w = (rng.random(d).astype(np.float32) + 0.5)
    xd = torch.from_numpy(x).to(DEV, torch.bfloat16)
    wd = torch.from_numpy(w).to(DEV, torch.bfloat16)
    out = torch.empty_like(xd)
    ops.rmsnorm(out, xd, wd, 1e-5)
    ref = orc.rmsnorm(xd.float().cpu().numpy(), wd.float().cpu().numpy(), 1e-5)
    np.testing.assert_allclose(out.float().cpu().numpy(), ref, rtol=1e-2, atol=1e-2)
