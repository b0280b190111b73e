"""Gathered decode LoRA kernels (large adapter pools) through the C ABI against the oracle.

slx_lora_shrink (A rows of the batch's adapters bulk-copied to shared memory, x staged per token
pair) and slx_lora_expand with v_slot_stride 0 (columns per thread chosen by rank) together are
the BGMV of oracle/llama_lora.py::bgmv (reference batch -> adapter association,
/root/reference/pkg/src/slorasim/batching.py:99-105; unmerged LoRA).
Covered: mixed ranks {8, 16, 24, 64} in one launch (every rank / 8 code path of the expand),
adapters spanning several plan tiles (> LORA_TT tokens), tokens without an adapter (slot -1,
rows untouched bit-for-bit), interleaved output column layouts, bf16 and fp32 activations."""
import numpy as np
import pytest
import torch

from oracle.llama_lora import bgmv
from paper_2505_14468_b200 import ops

pytestmark = pytest.mark.gpu


def _pool(n_slots, ranks, d_in, d_outs, seed):
    g = torch.Generator().manual_seed(seed)
    A, B = [], []
    for t, d_out in enumerate(d_outs):
        A.append([(torch.randn(int(r), d_in, generator=g) / d_in ** 0.5).to(torch.bfloat16).cuda()
                  for r in ranks])
        B.append([(torch.randn(d_out, int(r), generator=g) * 0.05).to(torch.bfloat16).cuda()
                  for r in ranks])
    a_ptr = [torch.tensor([a.data_ptr() for a in A[t]], dtype=torch.int64, device="cuda")
             for t in range(len(d_outs))]
    b_ptr = [torch.tensor([b.data_ptr() for b in B[t]], dtype=torch.int64, device="cuda")
             for t in range(len(d_outs))]
    return A, B, a_ptr, b_ptr


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("d_in,n_tok", [(512, 24), (5120, 64), (1024, 37), (8192, 16)])
def test_gathered_shrink_expand_matches_oracle(dtype, d_in, n_tok):
    torch.manual_seed(0)
    rng = np.random.default_rng(d_in + n_tok)
    ranks = [8, 16, 24, 64, 8, 16, 64]
    ns, R = len(ranks), 64
    d_outs = [d_in, d_in // 2, d_in // 2]             # q, k, v-like widths
    A, B, a_ptr, b_ptr = _pool(ns, ranks, d_in, d_outs, seed=d_in)
    scale = torch.tensor([2.0 * r / r for r in ranks], dtype=torch.float32, device="cuda") * 0.5
    rank_t = torch.tensor(ranks, dtype=torch.int32, device="cuda")
    tok_slot = rng.integers(-1, ns, size=n_tok).astype(np.int32)
    tok_slot[: min(11, n_tok)] = 3          # one adapter over two plan tiles (> LORA_TT tokens)
    tok_slot[-1] = -1
    rng.shuffle(tok_slot)
    slot_d = torch.from_numpy(tok_slot).cuda()
    x = torch.randn(n_tok, d_in, device="cuda").to(dtype)
    width = sum(d_outs)
    y0 = torch.randn(n_tok, width, device="cuda").to(dtype)
    ws = torch.zeros(ops.lora_workspace_bytes(n_tok, ns, R, 3) + 256, dtype=torch.uint8, device="cuda")
    ops.lora_plan_tokens(slot_d, ns, ws)
    offs = [0, R, 2 * R]
    tg = ops.make_targets([(a_ptr[t], b_ptr[t], d_outs[t], sum(d_outs[:t]), d_outs[t], d_outs[t])
                           for t in range(3)])
    v = torch.full((n_tok, 3 * R), float("nan"), device="cuda")
    ops.lora_shrink(v, x, rank_t, R, tg, offs, ws)
    y = y0.clone()
    ops.lora_expand(y, v, rank_t, scale, R, tg, offs, ws, v_slot_stride=0)
    torch.cuda.synchronize()
    xf = x.float().cpu().numpy()
    vn = v.cpu().numpy()
    # shrink: v = x A^T for the tokens' adapters (unscaled, fp32)
    for t in range(n_tok):
        s = tok_slot[t]
        if s < 0:
            continue
        for k in range(3):
            ref = xf[t] @ A[k][s].float().cpu().numpy().T
            np.testing.assert_allclose(vn[t, offs[k]:offs[k] + ranks[s]], ref, rtol=1e-4, atol=1e-3)
    # expand: y = y0 + bgmv, one rounding to the activation dtype
    yn, y0n = y.float().cpu().numpy(), y0.float().cpu().numpy()
    col = 0
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    for k in range(3):
        do = d_outs[k]
        ref = bgmv(y0n[:, col:col + do], xf, [a.float().cpu().numpy() for a in A[k]],
                   [b.float().cpu().numpy() for b in B[k]], scale.cpu().numpy(), tok_slot)
        np.testing.assert_allclose(yn[:, col:col + do], ref, rtol=tol, atol=tol)
        col += do
    # tokens without an adapter: untouched bit-for-bit
    none = tok_slot < 0
    assert torch.equal(y[torch.from_numpy(none).cuda()], y0[torch.from_numpy(none).cuda()])


def test_gathered_expand_rank_paths_follow_sequential_order():
    """Every rank / 8 instantiation of the expand (columns per thread 8..1) matches a sequential
    fp32 chain over j with v pre-scaled (the fused slx_lora_delta's order) within one bf16 ulp."""
    d_in, n_tok, R = 256, 16, 64
    ranks = [8, 16, 24, 32, 40, 48, 56, 64]
    ns = len(ranks)
    d_out = 4096
    A, B, a_ptr, b_ptr = _pool(ns, ranks, d_in, [d_out], seed=3)
    scale = torch.full((ns,), 0.75, dtype=torch.float32, device="cuda")
    rank_t = torch.tensor(ranks, dtype=torch.int32, device="cuda")
    tok_slot = np.array([i % ns for i in range(n_tok)], dtype=np.int32)
    ws = torch.zeros(ops.lora_workspace_bytes(n_tok, ns, R, 1) + 256, dtype=torch.uint8, device="cuda")
    ops.lora_plan_tokens(torch.from_numpy(tok_slot).cuda(), ns, ws)
    tg = ops.make_targets([(a_ptr[0], b_ptr[0], d_out, 0, d_out, d_out)])
    v = torch.randn(n_tok, R, device="cuda")
    y0 = torch.randn(n_tok, d_out, device="cuda").to(torch.bfloat16)
    y = y0.clone()
    ops.lora_expand(y, v, rank_t, scale, R, tg, [0], ws, v_slot_stride=0)
    torch.cuda.synchronize()
    vs = (v.cpu().numpy() * np.float32(0.75)).astype(np.float32)
    ref = np.empty((n_tok, d_out), dtype=np.float32)
    for t in range(n_tok):
        s = tok_slot[t]
        b = B[0][s].float().cpu().numpy()
        d = np.zeros(d_out, dtype=np.float32)
        for j in range(ranks[s]):          # sequential single-precision fma order
            d = (d + vs[t, j] * b[:, j]).astype(np.float32)
        ref[t] = y0[t].float().cpu().numpy() + d
    got = y.float().cpu().numpy()
    want = torch.from_numpy(ref).to(torch.bfloat16).float().numpy()
    # numpy's separate multiply-add may differ from fmaf by one fp32 rounding: allow 1 bf16 ulp
    ulp = np.abs(want) * 2.0 ** -7 + 1e-30
    assert np.all(np.abs(got - want) <= ulp)
