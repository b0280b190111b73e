"""Parity at BASELINE config 2's sizes (Llama-2-7B widths, 32 r16 adapters on q,k,v,o, batch 64).

* Against the oracle: one decoder layer at the full 7B widths (hidden 4096, 32 heads x 128,
  ffn 11008, vocab 32000), every token of the batch on its own adapter slot drawn like the
  bench's, prefill + one decode step through the same kernels as the bench (stacked shrink,
  split-K consumers, fused expands, tensor-core attention); bf16 tolerance as in
  test_gpu_model.py.
* Size-independent properties of the full 32-layer step: run-to-run bit identity, and exact
  equivariance under a permutation of the batch (every kernel treats rows independently).
"""
import numpy as np
import pytest
import torch

from oracle.llama_lora import OracleModel
from paper_2505_14468_b200.config import LLAMA2_7B, BackboneConfig, LoraConfig, init_adapter, init_backbone
from paper_2505_14468_b200.model import MultiLoraModel

pytestmark = pytest.mark.gpu

BATCH, N_ADAPTERS, RANK = 64, 32, 16
# bf16 bar at the 7B widths (K = 4096 / 11008 accumulations of bf16-rounded activations):
# relative Frobenius error of the logits <= 1e-2, max abs error <= 0.1 (logit std ~1.3), and
# the argmax agrees wherever the oracle's top-1 / top-2 margin exceeds TAU.
REL_FRO, MAX_ABS, TAU = 1e-2, 0.1, 0.05


def _check(got, ref, layers: int = 1):
    """The one-layer bar, widened by sqrt(layers) for deeper stacks (independent bf16 rounding
    errors per layer add in quadrature); argmax flips where the margin > TAU never allowed."""
    k = float(np.sqrt(layers))
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    mx = float(np.abs(got - ref).max())
    top2 = np.sort(ref, axis=1)[:, -2:]
    sure = (top2[:, 1] - top2[:, 0]) > TAU
    flips = int(((got.argmax(1) != ref.argmax(1)) & sure).sum())
    assert rel <= REL_FRO * k and mx <= MAX_ABS * k and flips == 0, (rel, mx, flips)


def _tok_slots(seed=0, batch=BATCH):
    return np.random.default_rng(seed).integers(0, N_ADAPTERS, size=batch).astype(np.int64).tolist()


@pytest.mark.parametrize("batch", [BATCH, 128])
def test_config2_widths_one_layer_decode_matches_oracle(batch):
    """Batch 64 (the bench's) and 128 (the decode path's M = 128 stream-K GEMMs)."""
    cfg = BackboneConfig("7b-1layer", hidden=4096, layers=1, heads=32, kv_heads=32, head_dim=128,
                         ffn=11008, vocab=32000)
    lora = LoraConfig(RANK, 32.0, ("q", "k", "v", "o"))
    w = init_backbone(cfg, 21)
    ads = [init_adapter(cfg, lora, 21, a) for a in range(N_ADAPTERS)]
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=batch, max_ctx=32, n_slots=N_ADAPTERS,
                       max_rank=RANK, max_tokens=batch * 16)
    m.load_backbone(w)
    for a, ad in enumerate(ads):
        m.pool.load(a, ad, lora)
    rng = np.random.default_rng(3)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=16))) for _ in range(batch)]
    ids = _tok_slots(batch=batch)
    ids[5] = ids[17] = -1   # tokens without an adapter ride along
    seqs, pre = m.prefill(prompts, ids)
    toks = list(map(int, rng.integers(1, cfg.vocab, size=batch)))
    assert m._decode_fast(batch)
    got = m.decode(seqs, toks, ids).float().cpu().numpy()
    orc = OracleModel(cfg, w, ads, [lora.scale] * N_ADAPTERS, lora.targets)
    ref_pre = orc.prefill(prompts, ids)
    ref = orc.decode(list(range(batch)), toks, ids)
    _check(pre.float().cpu().numpy(), ref_pre)
    _check(got, ref)


def test_config2_full_step_deterministic_and_permutation_equivariant():
    cfg = LLAMA2_7B
    lora = LoraConfig(RANK, 32.0, ("q", "k", "v", "o"))
    ctx = 128
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=BATCH, max_ctx=ctx + 1,
                       n_slots=N_ADAPTERS, max_rank=RANK, max_tokens=BATCH)
    m.random_backbone(seed=0)
    for a in range(N_ADAPTERS):
        m.pool.load_random(a, lora, seed=1000 + a)
    g = torch.Generator(device=m.device).manual_seed(7)
    for l in range(cfg.layers):
        m.k_cache[l].normal_(generator=g)
        m.v_cache[l].normal_(generator=g)
    seqs = [m.alloc_seq() for _ in range(BATCH)]
    slots = _tok_slots()
    toks = torch.randint(1, cfg.vocab, (BATCH,), generator=g, device=m.device).tolist()

    def step(order):
        for s in seqs:
            m.seq_len[s] = ctx
        return m.decode([seqs[i] for i in order], [toks[i] for i in order],
                        [slots[i] for i in order]).float()

    ident = list(range(BATCH))
    a = step(ident)
    b = step(ident)
    assert torch.equal(a, b)   # run-to-run bit identity (deterministic reductions)
    perm = np.random.default_rng(1).permutation(BATCH).tolist()
    c = step(perm)
    assert torch.equal(c, a[perm])   # rows are independent in every kernel
    assert torch.isfinite(a).all()


def test_13b_widths_one_layer_decode_matches_oracle():
    """The 13B widths (hidden 5120, 40 heads, ffn 13824: the one-CTA-per-token RMSNorm, 20-tile
    projections) through the same decode path, mixed ranks {8, 16} on q,k,v,o."""
    cfg = BackboneConfig("13b-1layer", hidden=5120, layers=1, heads=40, kv_heads=40, head_dim=128,
                         ffn=13824, vocab=32000)
    loras = [LoraConfig(16, 32.0, ("q", "k", "v", "o")), LoraConfig(8, 16.0, ("q", "k", "v", "o"))]
    w = init_backbone(cfg, 31)
    ads = [init_adapter(cfg, loras[a % 2], 31, a) for a in range(8)]
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=48, max_ctx=40, n_slots=8,
                       max_rank=16, max_tokens=48 * 24)
    m.load_backbone(w)
    for a, ad in enumerate(ads):
        m.pool.load(a, ad, loras[a % 2])
    rng = np.random.default_rng(4)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=int(rng.integers(1, 24)))))
               for _ in range(48)]
    ids = [int(i) for i in rng.integers(-1, 8, size=48)]
    seqs, pre = m.prefill(prompts, ids)
    toks = list(map(int, rng.integers(1, cfg.vocab, size=48)))
    got = m.decode(seqs, toks, ids).float().cpu().numpy()
    orc = OracleModel(cfg, w, ads, [loras[a % 2].scale for a in range(8)], loras[0].targets)
    ref_pre = orc.prefill(prompts, ids)
    ref = orc.decode(list(range(48)), toks, ids)
    _check(pre.float().cpu().numpy(), ref_pre)
    _check(got, ref)


def _pool_model(cfg, w, used, n_slots, max_rank, max_seqs, max_ctx, max_tokens, seed,
                decode_lora="auto"):
    """A model whose pool holds the oracle-known adapters ``used`` {slot: (LoraConfig, dict)}
    and seeded device-random adapters of ranks {8, 16, 64} in every other slot."""
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=max_seqs, max_ctx=max_ctx,
                       n_slots=n_slots, max_rank=max_rank, max_tokens=max_tokens,
                       decode_lora=decode_lora)
    m.load_backbone(w)
    ranks = np.random.default_rng(seed).choice([8, 16, 64], size=n_slots)
    for s in range(n_slots):
        if s in used:
            m.pool.load(s, used[s][1], used[s][0])
        else:
            m.pool.load_random(s, LoraConfig(int(ranks[s]), 2.0 * ranks[s]), seed=500 + s)
    return m


def test_config3_shape_one_layer_prefill_and_decode_match_oracle():
    """BASELINE config 3's shape, one layer: 13B widths (hidden 5120, 40 x 128 heads, ffn
    13824), a 128-slot pool of mixed ranks {8, 16, 64}, three 2048-token causal prompts (a
    rank-64 adapter, a rank-16 adapter, no adapter) through the bench's prefill path (LoRA
    folded into the tcgen05 backbone GEMMs, grouped tcgen05 shrink, flash prefill), and the
    SGMV path without the fold; then one decode step through the gathered-shrink decode path
    (the pool is too large to stack).  Logits of every 64th position vs the fp32 oracle."""
    cfg = BackboneConfig("13b-1layer", hidden=5120, layers=1, heads=40, kv_heads=40, head_dim=128,
                         ffn=13824, vocab=32000)
    L, n_slots = 2048, 128
    w = init_backbone(cfg, 41)
    lo64, lo16 = LoraConfig(64, 128.0, ("q", "k", "v", "o")), LoraConfig(16, 32.0, ("q", "k", "v", "o"))
    ad64, ad16 = init_adapter(cfg, lo64, 41, 0), init_adapter(cfg, lo16, 41, 1)
    used = {77: (lo64, ad64), 5: (lo16, ad16)}
    rng = np.random.default_rng(42)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=L))) for _ in range(3)]
    ids = [77, 5, -1]
    toks = list(map(int, rng.integers(1, cfg.vocab, size=3)))
    # oracle: adapters renumbered 0 (r64), 1 (r16)
    orc = OracleModel(cfg, w, [ad64, ad16], [lo64.scale, lo16.scale], lo64.targets, max_pos=L + 8)
    oid = {77: 0, 5: 1, -1: -1}
    for _ in range(3):
        orc.kv.append([(np.zeros((0, 40, 128), np.float32), np.zeros((0, 40, 128), np.float32))])
    tokens = np.concatenate([np.asarray(p) for p in prompts])
    positions = np.tile(np.arange(L), 3)
    indptr = np.array([0, L, 2 * L, 3 * L])
    h = orc._forward(tokens, positions, indptr, np.array([oid[i] for i in ids]), [0, 1, 2])
    rows = np.arange(0, 3 * L, 64)
    rows[-1] = 3 * L - 1
    ref_pre = orc.logits(h[rows])
    ref_dec = orc.decode([0, 1, 2], toks, [oid[i] for i in ids])
    for fold in (True, False):
        m = _pool_model(cfg, w, used, n_slots, 64, 4, L + 8, 3 * L, 41)
        assert m.decode_lora == "gather" and not m.stack
        m.lora_fold = fold
        seqs = [m.alloc_seq() for _ in range(3)]
        dev = m.device
        i32 = lambda v: torch.tensor(np.asarray(v), dtype=torch.int32, device=dev)  # noqa: E731
        slot = np.repeat(np.asarray(ids), L)
        got = m.forward(i32(tokens), i32(positions), i32(np.repeat(seqs, L)), i32(slot),
                        torch.tensor(rows, dtype=torch.int64, device=dev),
                        segments=m.segments_of(positions, np.repeat(seqs, L)))
        _check(got.float().cpu().numpy(), ref_pre)
        for s in seqs:
            m.seq_len[s] = L
        dec = m.decode(seqs, toks, ids)
        _check(dec.float().cpu().numpy(), ref_dec)
        del m
        torch.cuda.empty_cache()


def test_7b_widths_four_layer_decode_matches_oracle():
    """Error growth across layers: four decoder layers at the 7B widths, batch 64 on 32 r16
    adapters (the bench's slot draw, two tokens without adapter), a 16-token prefill and
    three decode steps through the stacked decode path AND the gathered-shrink path, each
    step's logits vs the fp32 oracle at the one-layer bar widened by sqrt(4) (bf16 rounding
    of four layers' activations accumulates; no argmax flip above TAU)."""
    cfg = BackboneConfig("7b-4layer", hidden=4096, layers=4, heads=32, kv_heads=32, head_dim=128,
                         ffn=11008, vocab=32000)
    lora = LoraConfig(RANK, 32.0, ("q", "k", "v", "o"))
    w = init_backbone(cfg, 23)
    ads = [init_adapter(cfg, lora, 23, a) for a in range(N_ADAPTERS)]
    rng = np.random.default_rng(6)
    prompts = [list(map(int, rng.integers(1, cfg.vocab, size=16))) for _ in range(BATCH)]
    ids = _tok_slots()
    ids[3] = ids[40] = -1
    steps = [list(map(int, rng.integers(1, cfg.vocab, size=BATCH))) for _ in range(3)]
    orc = OracleModel(cfg, w, ads, [lora.scale] * N_ADAPTERS, lora.targets)
    ref_pre = orc.prefill(prompts, ids)
    refs = [orc.decode(list(range(BATCH)), t, ids) for t in steps]
    for mode in ("stacked", "gather"):
        m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=BATCH, max_ctx=32,
                           n_slots=N_ADAPTERS, max_rank=RANK, max_tokens=BATCH * 16,
                           decode_lora=mode)
        m.load_backbone(w)
        for a, ad in enumerate(ads):
            m.pool.load(a, ad, lora)
        assert m._decode_fast(BATCH)
        seqs, pre = m.prefill(prompts, ids)
        _check(pre.float().cpu().numpy(), ref_pre, layers=4)
        for t, ref in zip(steps, refs):
            _check(m.decode(seqs, t, ids).float().cpu().numpy(), ref, layers=4)
        del m
        torch.cuda.empty_cache()
