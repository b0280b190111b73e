"""CPU: FlushDecisions -> adapter-segmented mixed batches."""

import numpy as np

from paper_2505_14468_b200.batching import FlushDecision
from paper_2505_14468_b200.segments import (Request, build_decode, build_mixed, build_prefill,
                                             group_by_gpu)


def _reqs():
    rs = [Request(i, f"f{i % 3}", list(range(10 * i + 1, 10 * i + 1 + (i % 4) + 1)), 4) for i in range(7)]
    for i, r in enumerate(rs):
        r.seq = i
        r.adapter_slot = [2, -1, 0][i % 3]
    return rs


def test_prefill_segments_grouped_by_adapter():
    rs = _reqs()
    seq_len = [0] * 8
    seq_len[3] = 5          # a continuing sequence starts at its cached length
    b = build_prefill(rs, seq_len)
    assert b.n_tokens == sum(len(r.prompt) for r in rs)
    assert list(b.seg_slot) == sorted(b.seg_slot.tolist())     # grouped by adapter slot
    for s, r in enumerate(b.requests):
        lo, hi = b.seg_indptr[s], b.seg_indptr[s + 1]
        assert b.tokens[lo:hi].tolist() == r.prompt
        assert (b.seq[lo:hi] == r.seq).all() and (b.slot[lo:hi] == r.adapter_slot).all()
        assert b.pos[lo:hi].tolist() == list(range(seq_len[r.seq], seq_len[r.seq] + hi - lo))
        assert b.logit_rows[s] == hi - 1


def test_decode_one_token_per_sequence():
    rs = _reqs()
    for r in rs:
        r.generated = [r.request_id + 100]
    seq_len = list(range(8))
    b = build_decode(rs, seq_len)
    assert b.tokens.tolist() == [r.request_id + 100 for r in rs]
    assert b.pos.tolist() == [seq_len[r.seq] for r in rs]
    assert b.slot.tolist() == [r.adapter_slot for r in rs]
    assert b.seg_indptr.tolist() == list(range(len(rs) + 1))


def test_group_by_gpu():
    ds = [FlushDecision("a", "g0", (1,), "fill"), FlushDecision("b", "g1", (2,), "expire"),
          FlushDecision("c", "g0", (3, 4), "margin", 1.0)]
    g = group_by_gpu(ds)
    assert [d.function_id for d in g["g0"]] == ["a", "c"] and len(g["g1"]) == 1


def test_mixed_round_prefill_then_one_token_per_running_sequence():
    rs = _reqs()
    new, running = rs[:4], rs[4:]
    for r in running:
        r.generated = [r.request_id + 100]
    seq_len = [0] * 8
    for r in running:
        seq_len[r.seq] = 7 + r.seq
    b, n = build_mixed(new, running, seq_len)
    p = build_prefill(new, seq_len)
    d = build_decode(running, seq_len)
    assert n == len(new) and b.requests[:n] == p.requests and b.requests[n:] == running
    T = p.n_tokens
    assert b.n_tokens == T + len(running)
    assert b.tokens.tolist() == p.tokens.tolist() + d.tokens.tolist()
    assert b.pos[T:].tolist() == [seq_len[r.seq] for r in running]     # cached-prefix segments
    assert b.seg_indptr.tolist() == p.seg_indptr.tolist() + [T + i + 1 for i in range(len(running))]
    assert b.logit_rows.tolist() == p.logit_rows.tolist() + [T + i for i in range(len(running))]
    assert b.seg_slot.tolist() == p.seg_slot.tolist() + [r.adapter_slot for r in running]


def _prefill_plan_loops(segments, heads, bq):
    """The flash plan as straight loops (the vectorised ops.prefill_plan must equal it)."""
    tiles, items = [], []
    for tok0, n, seq, pos0 in segments:
        ids = []
        for q in range(0, n, bq):
            ids.append(len(tiles))
            tiles.append((tok0 + q, min(bq, n - q), seq, pos0 + q))
        pairs = [(ids[k + 1], ids[k]) if k + 1 < len(ids) else (ids[k], -1)
                 for k in range(0, len(ids), 2)]
        for h in range(heads):
            items += [(a, b, h, 0) for a, b in pairs]

    def cost(it):
        a, b = tiles[it[0]], (tiles[it[1]] if it[1] >= 0 else None)
        return -(-(a[3] + a[1]) // 64) + (-(-(b[3] + b[1]) // 64) if b else 0)
    items.sort(key=lambda it: -cost(it))
    return tiles, items


def test_flash_prefill_plan_matches_loops():
    from paper_2505_14468_b200.ops import prefill_plan
    rng = np.random.default_rng(3)
    for trial in range(30):
        segs, tok = [], 0
        for s in range(int(rng.integers(1, 40))):
            n = int(rng.choice([1, 1, 5, 64, 127, 128, 129, 300, 2048]))
            segs.append((tok, n, s, int(rng.integers(0, 200)) if rng.random() < 0.5 else 0))
            tok += n
        heads = int(rng.choice([1, 4, 32]))
        t, it = prefill_plan(segs, heads, "cpu", bq=128)
        rt, ri = _prefill_plan_loops(segs, heads, 128)
        assert t.tolist() == [list(x) for x in rt]
        assert it.tolist() == [list(x) for x in ri]


def test_segments_of_runs_match_loop():
    from paper_2505_14468_b200.model import MultiLoraModel
    rng = np.random.default_rng(5)
    for _ in range(50):
        pos, seq = [], []
        for s in range(int(rng.integers(1, 12))):
            n = int(rng.integers(1, 9))
            p0 = int(rng.integers(0, 30))
            q = int(rng.integers(0, 4))
            pos += list(range(p0, p0 + n))
            seq += [q] * n
        ref, start = [], 0
        for i in range(1, len(pos) + 1):
            if i == len(pos) or seq[i] != seq[start] or pos[i] != pos[i - 1] + 1:
                ref.append((start, i - start, seq[start], pos[start]))
                start = i
        assert MultiLoraModel.segments_of(np.array(pos, np.int32), np.array(seq, np.int32)) == ref
    assert MultiLoraModel.segments_of(np.zeros(0, np.int32), np.zeros(0, np.int32)) == []
