"""GPU: end-to-end config-1 parity of the multi-LoRA runtime.

* fp32 parity mode: greedy tokens bit-exact vs the oracle AND the transformers golden.
* bf16 mode: teacher-forced logits within rtol 2e-2 (atol 2e-2 on |logit| ~ 1.5) of the
  fp32 oracle, and greedy argmax agreement wherever the oracle's top-1/top-2 margin
  exceeds TAU (bf16 rounding can legitimately flip near-ties).
"""

import numpy as np
import pytest
import torch

from oracle.llama_lora import OracleModel
from paper_2505_14468_b200.config import TINY, TINY_LORA, LoraConfig, init_adapter, init_backbone
from paper_2505_14468_b200.model import MultiLoraModel

pytestmark = pytest.mark.gpu
TAU = 0.05          # logit margin above which bf16 must agree with the fp32 oracle
BF16_RTOL = 2e-2
BF16_ATOL = 2e-2


def _setup(golden, dtype, targets=TINY_LORA.targets):
    cfg = TINY
    lora = LoraConfig(TINY_LORA.rank, TINY_LORA.alpha, targets)
    seed = int(golden["seed"])
    w = init_backbone(cfg, seed)
    ads = [init_adapter(cfg, lora, seed, a) for a in range(int(golden["n_adapters"]))]
    m = MultiLoraModel(cfg, dtype=dtype, max_seqs=16, max_ctx=128, lora_targets=targets,
                       n_slots=8, max_rank=16, max_tokens=1024)
    m.load_backbone(w)
    for a, ad in enumerate(ads):
        m.pool.load(a, ad, lora)
    ip = golden["prompt_indptr"]
    prompts = [list(map(int, golden["prompt_flat"][ip[i]:ip[i + 1]])) for i in range(len(ip) - 1)]
    return m, w, ads, lora, prompts


def test_fp32_parity_greedy_tokens_bit_exact(golden):
    m, w, ads, lora, prompts = _setup(golden, torch.float32)
    toks = m.generate(prompts, list(map(int, golden["adapter_ids"])), int(golden["n_new"]))
    assert np.array_equal(toks, golden["tokens"]), np.argwhere(toks != golden["tokens"])[:5]


def test_bf16_teacher_forced_logits(golden):
    m, w, ads, lora, prompts = _setup(golden, torch.bfloat16)
    toks = golden["tokens"]
    adapter_ids = list(map(int, golden["adapter_ids"]))
    # teacher forcing: prefill prompt + golden continuation, logits at every generated position
    seqs = [p + list(map(int, toks[i, :-1])) for i, p in enumerate(prompts)]
    orc = OracleModel(TINY, w, ads, [lora.scale] * len(ads), lora.targets)
    flips, checked = 0, 0
    for i, s in enumerate(seqs):
        dev = m.device
        L = len(s)
        t = torch.tensor(s, dtype=torch.int32, device=dev)
        pos = torch.arange(L, dtype=torch.int32, device=dev)
        sq = torch.full((L,), 0, dtype=torch.int32, device=dev)
        sl = torch.full((L,), adapter_ids[i], dtype=torch.int32, device=dev)
        got = m.forward(t, pos, sq, sl).cpu().numpy()[len(prompts[i]) - 1:]
        ref = orc.teacher_forced(s, adapter_ids[i])[len(prompts[i]) - 1:]
        np.testing.assert_allclose(got, ref, rtol=BF16_RTOL, atol=BF16_ATOL)
        part = np.partition(ref, -2, axis=-1)
        margin = part[:, -1] - part[:, -2]
        sure = margin > TAU
        checked += int(sure.sum())
        flips += int((np.argmax(got, -1)[sure] != np.argmax(ref, -1)[sure]).sum())
    assert checked > 100
    assert flips == 0


def test_bf16_greedy_agrees_where_margin_large(golden):
    m, w, ads, lora, prompts = _setup(golden, torch.bfloat16)
    toks = m.generate(prompts, list(map(int, golden["adapter_ids"])), int(golden["n_new"]))
    gold = golden["tokens"]
    margin = golden["margin"]
    # compare up to (and including) the first position of each request whose margin < TAU
    for r in range(gold.shape[0]):
        for s in range(gold.shape[1]):
            if margin[r, s] < TAU:
                break
            assert toks[r, s] == gold[r, s], (r, s)


def test_fp32_parity_all_linear_targets(golden):
    """LoRA on every projection (gate/up through the blocked layout, down with padded ffn)."""
    targets = ("q", "k", "v", "o", "gate", "up", "down")
    m, w, ads, lora, prompts = _setup(golden, torch.float32, targets)
    orc = OracleModel(TINY, w, ads, [lora.scale] * len(ads), targets)
    ids = list(map(int, golden["adapter_ids"]))[:6]
    ref, _ = orc.generate(prompts[:6], ids, 8)
    got = m.generate(prompts[:6], ids, 8)
    assert np.array_equal(got, ref)


def test_bf16_all_linear_targets_logits(golden):
    targets = ("q", "k", "v", "o", "gate", "up", "down")
    m, w, ads, lora, prompts = _setup(golden, torch.bfloat16, targets)
    orc = OracleModel(TINY, w, ads, [lora.scale] * len(ads), targets)
    ids = list(map(int, golden["adapter_ids"]))[:6]
    ref = orc.prefill(prompts[:6], ids)
    seqs, got = m.prefill(prompts[:6], ids)
    np.testing.assert_allclose(got.cpu().numpy(), ref, rtol=BF16_RTOL, atol=BF16_ATOL)


def test_bf16_stacked_decode_shrink_matches_sgmv_path(golden):
    """Decode LoRA with the shrink inside the projection GEMM (stacked A rows, fp32 side
    output) + expand kernel == the shrink/expand kernel path == the oracle; mixed ranks."""
    cfg = TINY
    seed = int(golden["seed"])
    w = init_backbone(cfg, seed)
    loras = [LoraConfig(8, 16.0), LoraConfig(16, 8.0), LoraConfig(8, 16.0), LoraConfig(16, 32.0)]
    ads = [init_adapter(cfg, lo, seed, a) for a, lo in enumerate(loras)]
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=6, max_rank=16,
                       max_tokens=512)
    m.load_backbone(w)
    for a, (ad, lo) in enumerate(zip(ads, loras)):
        m.pool.load(a, ad, lo)
    prompts = [[5, 9, 200, 31], [7, 7, 7], [100, 2, 3, 4, 5], [9]]
    ids = [0, 1, 3, 2]
    seqs, _ = m.prefill(prompts, ids)
    toks = [11, 12, 13, 14]
    got = {}
    for stacked, fuse in ((True, True), (True, False), (False, False)):
        m.use_stacked_decode, m.fuse_expand = stacked, fuse
        for s_ in seqs:
            m.seq_len[s_] = len(prompts[seqs.index(s_)])
        got[(stacked, fuse)] = m.decode(seqs, toks, ids).cpu().numpy()
    m.fuse_expand = True
    # the expand fused into attention / post-norm rounds exactly like the expand kernel
    np.testing.assert_array_equal(got[(True, True)], got[(True, False)])
    got[True], got[False] = got[(True, True)], got[(False, False)]
    np.testing.assert_allclose(got[True], got[False], rtol=1e-2, atol=1e-2)
    orc = OracleModel(cfg, w, ads, [lo.scale for lo in loras], loras[0].targets)
    orc.prefill(prompts, ids)
    ref = orc.decode(list(range(4)), toks, ids)
    np.testing.assert_allclose(got[True], ref, rtol=BF16_RTOL, atol=BF16_ATOL)
    # gathered decode shrink (slx_lora_shrink + fused expands, v_slot_stride 0) == stacked
    mg = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=6, max_rank=16,
                        max_tokens=512, decode_lora="gather")
    mg.load_backbone(w)
    for a, (ad, lo) in enumerate(zip(ads, loras)):
        mg.pool.load(a, ad, lo)
    sg, _ = mg.prefill(prompts, ids)
    gg = mg.decode(sg, toks, ids).cpu().numpy()
    np.testing.assert_allclose(gg, got[True], rtol=1e-2, atol=1e-2)
    np.testing.assert_allclose(gg, ref, rtol=BF16_RTOL, atol=BF16_ATOL)
    # eviction zeroes the stacked rows: slot 1 then behaves like the bare backbone
    m.use_stacked_decode = True
    m.pool.evict(1)
    for s_ in seqs:
        m.seq_len[s_] = len(prompts[seqs.index(s_)])
    ev = m.decode(seqs, toks, [0, -1, 3, 2]).cpu().numpy()
    for s_ in seqs:
        m.seq_len[s_] = len(prompts[seqs.index(s_)])
    ev2 = m.decode(seqs, toks, [0, 1, 3, 2]).cpu().numpy()   # slot 1 evicted: rank 0
    np.testing.assert_allclose(ev[1], ev2[1], rtol=1e-2, atol=1e-2)


def test_bf16_prefill_lora_fold_matches_oracle(monkeypatch):
    """Prefill with the LoRA expand folded into the backbone qkv / o GEMMs (one extra K block
    per segment-aligned tile) == the separate shrink/expand SGMV path == oracle; mixed ranks,
    a prompt without adapter, a segment that is not a multiple of 128 tokens."""
    from paper_2505_14468_b200.config import BackboneConfig
    cfg = BackboneConfig("small128", hidden=512, layers=2, heads=4, kv_heads=2, head_dim=128,
                         ffn=1024, vocab=1000)
    w = init_backbone(cfg, 5)
    loras = [LoraConfig(8, 16.0), LoraConfig(64, 32.0), LoraConfig(16, 16.0)]
    ads = [init_adapter(cfg, lo, 5, a) for a, lo in enumerate(loras)]
    rng = np.random.default_rng(9)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=L))) for L in (256, 128, 200, 384)]
    ids = [1, 0, -1, 2]
    out = {}
    for fold in (True, False):
        m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=512, n_slots=4,
                           max_rank=64, max_tokens=1024)
        m.lora_fold = fold
        m.load_backbone(w)
        for a, (ad, lo) in enumerate(zip(ads, loras)):
            m.pool.load(a, ad, lo)
        _, lg = m.prefill(prompts, ids)
        out[fold] = lg.cpu().numpy()
    np.testing.assert_allclose(out[True], out[False], rtol=2e-2, atol=2e-2)
    orc = OracleModel(cfg, w, ads, [lo.scale for lo in loras], loras[0].targets)
    ref = orc.prefill(prompts, ids)
    np.testing.assert_allclose(out[True], ref, rtol=BF16_RTOL, atol=BF16_ATOL)


def test_bf16_decode_splitk_consumer_matches_oracle():
    """Decode with the o / down projections as split-K pieces reduced by the following RMSNorm
    (residual epilogue, o-LoRA v and delta fused there) == the GEMM-side reduction == oracle."""
    from paper_2505_14468_b200.config import BackboneConfig
    cfg = BackboneConfig("w2048", hidden=2048, layers=2, heads=16, kv_heads=16, head_dim=128,
                         ffn=2048, vocab=1000)
    w = init_backbone(cfg, 11)
    loras = [LoraConfig(16, 32.0), LoraConfig(8, 16.0), LoraConfig(16, 8.0)]
    ads = [init_adapter(cfg, lo, 11, a) for a, lo in enumerate(loras)]
    prompts = [[5, 9, 200, 31], [7, 7, 7], [100, 2, 3, 4, 5], [9], [44, 45]]
    ids = [0, 1, 2, -1, 1]
    toks = [11, 12, 13, 14, 15]
    out = {}
    for sk in (True, False):
        m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=4,
                           max_rank=16, max_tokens=256)
        m.splitk_consumer = sk
        m.load_backbone(w)
        for a, (ad, lo) in enumerate(zip(ads, loras)):
            m.pool.load(a, ad, lo)
        seqs, _ = m.prefill(prompts, ids)
        out[sk] = m.decode(seqs, toks, ids).cpu().numpy()
    # the split-K consumer norm == the GEMM-side reduction
    np.testing.assert_allclose(out[True], out[False], rtol=2e-2, atol=2e-2)
    orc = OracleModel(cfg, w, ads, [lo.scale for lo in loras], loras[0].targets)
    orc.prefill(prompts, ids)
    ref = orc.decode(list(range(len(prompts))), toks, ids)
    np.testing.assert_allclose(out[True], ref, rtol=BF16_RTOL, atol=BF16_ATOL)


@pytest.mark.parametrize("small_lora", ["stacked", "gather"])
def test_bf16_prefill_tc_path_matches_oracle(small_lora):
    """Prefill with the tensor-core paths on a head_dim-128 GQA model with mixed adapter ranks
    {8,16,64} == SIMT paths == oracle.  The short ragged segments make the LoRA fold decline,
    so the LoRA runs as the small-batch path: the stacked shrink as the projection GEMM's side
    output + expand kernel, or the gathered shrink / expand kernels."""
    from paper_2505_14468_b200.config import BackboneConfig
    cfg = BackboneConfig("small128", hidden=512, layers=2, heads=4, kv_heads=2, head_dim=128,
                         ffn=1024, vocab=1000)
    w = init_backbone(cfg, 3)
    loras = [LoraConfig(8, 16.0), LoraConfig(64, 32.0), LoraConfig(16, 16.0)]
    ads = [init_adapter(cfg, lo, 3, a) for a, lo in enumerate(loras)]
    rng = np.random.default_rng(5)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=L))) for L in (300, 7, 129, 64, 1)]
    ids = [1, 0, 2, 1, -1]
    out = {}
    for tc in (True, False):
        m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=512, n_slots=4,
                           max_rank=64, max_tokens=1024)
        m.use_tc_sgmv = tc
        m.prefill_small_lora = small_lora
        m.load_backbone(w)
        for a, (ad, lo) in enumerate(zip(ads, loras)):
            m.pool.load(a, ad, lo)
        _, lg = m.prefill(prompts, ids)
        out[tc] = lg.cpu().numpy()
    np.testing.assert_allclose(out[True], out[False], rtol=2e-2, atol=2e-2)
    orc = OracleModel(cfg, w, ads, [lo.scale for lo in loras], loras[0].targets)
    ref = orc.prefill(prompts, ids)
    np.testing.assert_allclose(out[True], ref, rtol=BF16_RTOL, atol=BF16_ATOL)


def test_bf16_bare_backbone_decode_takes_the_splitk_path():
    """A model without LoRA targets decodes through the same split-K path as the LoRA model
    (bench's bare-backbone reference for the LoRA marginal) and agrees with the LoRA model on
    tokens that carry no adapter."""
    from paper_2505_14468_b200.config import BackboneConfig
    cfg = BackboneConfig("w2048", hidden=2048, layers=2, heads=16, kv_heads=16, head_dim=128,
                         ffn=2048, vocab=1000)
    w = init_backbone(cfg, 5)
    lo = LoraConfig(16, 32.0)
    prompts, toks = [[5, 9, 200, 31], [7, 7, 7], [44, 45]], [11, 12, 13]
    out = {}
    for targets in ((), lo.targets):
        m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=4, max_ctx=64, n_slots=2,
                           max_rank=16, max_tokens=128, lora_targets=targets)
        m.load_backbone(w)
        if targets:
            m.pool.load(0, init_adapter(cfg, lo, 5, 0), lo)
        ids = [-1, -1, -1]
        seqs, _ = m.prefill(prompts, ids)
        out[bool(targets)] = m.decode(seqs, toks, ids).cpu().numpy()
    np.testing.assert_allclose(out[False], out[True], rtol=2e-2, atol=2e-2)
