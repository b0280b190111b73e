"""The decode layer chain (slx_decode_chain: o -> post-norm -> gate/up -> down -> input norm ->
q/k/v -> reduction as ONE persistent launch per layer, grid barriers between the phases).

Its pieces, reductions and norms follow the separate kernels' arithmetic exactly (same K ranges,
piece order, summation trees and roundings), so the decode logits must be BIT-identical to the
separate-kernel step (`use_chain = False`), which the oracle tests pin (test_gpu_fullsize.py,
test_gpu_model.py run the chain by default).  Also: graph capture, batch sizes below 64, and
the barrier counters left zeroed."""
import numpy as np
import pytest
import torch

from paper_2505_14468_b200 import ops
from paper_2505_14468_b200.config import TINY, BackboneConfig, LoraConfig
from paper_2505_14468_b200.engine import DecodeGraph
from paper_2505_14468_b200.model import MultiLoraModel

pytestmark = pytest.mark.gpu

CFG_7B2 = BackboneConfig("7b-2layer", hidden=4096, layers=2, heads=32, kv_heads=32, head_dim=128,
                         ffn=11008, vocab=32000)


def _model(cfg, n_slots, rank, batch, ctx=40, seed=0):
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=batch, max_ctx=ctx, n_slots=n_slots,
                       max_rank=rank, max_tokens=batch * 16)
    m.random_backbone(seed=seed)
    lora = LoraConfig(rank, 2.0 * rank, ("q", "k", "v", "o"))
    for a in range(n_slots):
        m.pool.load_random(a, lora, seed=100 + a)
    return m


def _prefill(m, batch, slots, plen=12, seed=1):
    rng = np.random.default_rng(seed)
    prompts = [list(map(int, rng.integers(1, m.cfg.vocab, size=plen))) for _ in range(batch)]
    seqs, _ = m.prefill(prompts, slots)
    return seqs, list(map(int, rng.integers(1, m.cfg.vocab, size=batch)))


def _decode_both(m, seqs, toks, slots):
    assert m._chain_ok(len(seqs))
    m.use_chain = True
    a = m.decode(seqs, toks, slots).clone()
    for s in seqs:   # decode() advanced the lengths: rewind, decode the same position again
        m.seq_len[s] -= 1
    m.use_chain = False
    b = m.decode(seqs, toks, slots).clone()
    m.use_chain = True
    return a, b


@pytest.mark.parametrize("batch", [64, 17, 1])
def test_chain_bit_identical_to_separate_kernels_7b_widths(batch):
    m = _model(CFG_7B2, 32, 16, 64)
    rng = np.random.default_rng(batch)
    slots = rng.integers(0, 32, size=batch).tolist()
    if batch > 4:
        slots[1] = slots[3] = -1   # tokens without an adapter ride along
    seqs, toks = _prefill(m, batch, slots)
    a, b = _decode_both(m, seqs, toks, slots)
    assert torch.isfinite(a).all()
    assert torch.equal(a, b), float((a - b).abs().max())
    assert int(m.chain_sync[:32].abs().sum()) == 0   # barrier counters left zeroed


def test_chain_bit_identical_tiny_and_bare_backbone():
    m = _model(TINY, 4, 8, 16)
    slots = [0, 1, 2, 3, -1, 0, 1, 2, 3, -1, 3, 2, 1, 0, 0, 1]
    seqs, toks = _prefill(m, 16, slots)
    a, b = _decode_both(m, seqs, toks, slots)
    assert torch.equal(a, b)
    bare = MultiLoraModel(TINY, dtype=torch.bfloat16, max_seqs=16, max_ctx=40, n_slots=4,
                          max_rank=8, lora_targets=())
    bare.random_backbone(seed=3)
    seqs, toks = _prefill(bare, 16, [-1] * 16)
    a, b = _decode_both(bare, seqs, toks, [-1] * 16)
    assert torch.equal(a, b)


def test_chain_graph_replay_matches_eager_and_launch_count():
    m = _model(CFG_7B2, 32, 16, 64)
    slots = np.random.default_rng(0).integers(0, 32, size=64).tolist()
    seqs, toks = _prefill(m, 64, slots)
    pos = m.seq_len[seqs[0]]
    dg = DecodeGraph(m, seqs, slots, fixed_pos=pos)
    dg.tok.copy_(torch.tensor(toks, dtype=torch.int32, device=m.device))
    dg.capture()
    # embedding + plan + head chain + per layer (attention + chain) + lm_head + argmax
    assert dg.kernels_per_step == 2 + 1 + 2 * m.cfg.layers + 1 + 1
    dg.replay()
    torch.cuda.synchronize()
    g = dg.logits.clone()
    for _ in range(3):
        dg.replay()
    torch.cuda.synchronize()
    assert torch.equal(g, dg.logits)   # run-to-run bit identity through the barriers
    e = m.forward(dg.tok, dg.pos, dg.seq, dg.slot, decode=True)
    assert torch.equal(g, e)
    assert int(m.chain_sync[:32].abs().sum()) == 0


def test_chain_rejects_shapes_outside_its_envelope():
    m = _model(TINY, 4, 8, 16)
    x = torch.zeros(65, TINY.hidden, dtype=torch.bfloat16, device=m.device)
    ph = ops.chain_norm(x, x, m.w["final_norm"], 1e-5)
    assert ops.chain_ctas([ph], 65) == 0          # M > 64
    assert ops.chain_ctas([ph], 64) > 0
    with pytest.raises(ValueError):
        ops.decode_chain([ph], 65, m.chain_sync)
