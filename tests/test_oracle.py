"""CPU: the oracle against the committed transformers-generated golden fixture."""

import numpy as np

from oracle.llama_lora import OracleModel, attention, bgmv, lora_delta, sgmv, top2_margin
from paper_2505_14468_b200.config import (
    TINY, TINY_LORA, init_adapter, init_backbone, round_to_bf16, synthetic_requests)

from golden.make_golden import weights_digest


def _tiny(golden):
    cfg, lora = TINY, TINY_LORA
    w = init_backbone(cfg, int(golden["seed"]))
    ads = [init_adapter(cfg, lora, int(golden["seed"]), a) for a in range(int(golden["n_adapters"]))]
    ip = golden["prompt_indptr"]
    prompts = [list(golden["prompt_flat"][ip[i]:ip[i + 1]]) for i in range(len(ip) - 1)]
    return cfg, lora, w, ads, prompts


def test_init_spec_is_pinned(golden):
    cfg, lora, w, ads, prompts = _tiny(golden)
    assert weights_digest(w) == str(golden["weights_sha256"])
    reqs = synthetic_requests(16, 4, cfg.vocab, int(golden["seed"]))
    assert [r.prompt for r in reqs] == prompts
    assert all(np.array_equal(round_to_bf16(v), v) for v in w.values())


def test_oracle_matches_transformers_golden(golden):
    cfg, lora, w, ads, prompts = _tiny(golden)
    m = OracleModel(cfg, w, ads, [lora.scale] * len(ads), lora.targets)
    toks, logits = m.generate(prompts, list(golden["adapter_ids"]), int(golden["n_new"]))
    assert np.array_equal(toks, golden["tokens"])            # bit-exact greedy tokens
    for (r, s), kl in zip(golden["kept_index"], golden["kept_logits"]):
        np.testing.assert_allclose(logits[r, s], kl, rtol=0, atol=1e-5)
    np.testing.assert_allclose(top2_margin(logits), golden["margin"], atol=1e-5)
    lg = logits.astype(np.float64)
    np.testing.assert_allclose(lg.sum(-1), golden["logit_sum"], rtol=1e-5, atol=1e-2)
    np.testing.assert_allclose((lg * lg).sum(-1), golden["logit_sumsq"], rtol=1e-5)


def test_lora_changes_output(golden):
    """Adapters are live: a request's tokens change if its adapter is dropped."""
    cfg, lora, w, ads, prompts = _tiny(golden)
    m = OracleModel(cfg, w, ads, [lora.scale] * len(ads), lora.targets)
    toks, _ = m.generate(prompts[:4], [-1] * 4, 8)
    assert not np.array_equal(toks, golden["tokens"][:4, :8])


def test_bgmv_sgmv_agree_with_per_token_loop():
    rng = np.random.default_rng(0)
    T, di, do, r, S = 37, 48, 40, 8, 5
    x = rng.standard_normal((T, di)).astype(np.float32)
    y = rng.standard_normal((T, do)).astype(np.float32)
    A = [rng.standard_normal((r, di)).astype(np.float32) for _ in range(S)]
    B = [rng.standard_normal((do, r)).astype(np.float32) for _ in range(S)]
    sc = [0.5 + a for a in range(S)]
    slot = rng.integers(-1, S, size=T)
    ref = y.copy()
    for t in range(T):
        if slot[t] >= 0:
            ref[t] += lora_delta(x[t:t + 1], A[slot[t]], B[slot[t]], sc[slot[t]])[0]
    np.testing.assert_allclose(bgmv(y, x, A, B, sc, slot), ref, rtol=1e-4, atol=1e-4)
    # segments: one run per slot in sorted order, including empty segments
    order = np.argsort(slot, kind="stable")
    seg_slot = np.arange(-1, S)
    indptr = np.concatenate([[0], np.cumsum([(slot == s).sum() for s in seg_slot])])
    out = sgmv(y[order], x[order], A, B, sc, indptr, seg_slot)
    np.testing.assert_allclose(out, ref[order], rtol=1e-4, atol=1e-4)


def test_attention_causal_and_gqa():
    rng = np.random.default_rng(1)
    q = rng.standard_normal((5, 4, 8)).astype(np.float32)
    k = rng.standard_normal((5, 2, 8)).astype(np.float32)
    v = rng.standard_normal((5, 2, 8)).astype(np.float32)
    out = attention(q, k, v, np.arange(5))
    # first query sees only key 0
    np.testing.assert_allclose(out[0, 0], v[0, 0], rtol=1e-6)
    np.testing.assert_allclose(out[0, 3], v[0, 1], rtol=1e-6)
