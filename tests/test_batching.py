"""CPU: the batcher mirror reproduces the reference's known-answer tests and, where the
reference is importable in this container, its exact decisions on random rounds."""

import math
import os
import random
import sys

import pytest

from paper_2505_14468_b200.batching import (
    BatchQueue, FlushDecision, batch_delay, deadline_margin, max_batch_size, predict_ttft,
    schedule_round)
from paper_2505_14468_b200.spec import ArtifactKind, ArtifactSpec, ConfigError, FunctionSpec

REF_SRC = "/root/reference/pkg/src"


def fn(fid="7b-chat", t0=500.0, alpha=100.0, slo=2500.0, kv=100_000_000):
    arts = (ArtifactSpec(ArtifactKind.ADAPTER_MODEL, 200_000_000, 100.0, 4.0),)
    return FunctionSpec(fid, arts, slo, t0, alpha, 10.0, kv, 800.0, backbone_id="llama7b")


def test_closed_forms_7b_profile():
    """tests/test_acceptance.py:85-92 of the reference."""
    f = fn()
    assert max_batch_size(f) == 21
    assert batch_delay(f, 5) == 1600.0
    assert predict_ttft(f, 5) == 900.0
    assert deadline_margin(f, 5, waited_ms=300.0, m=2) == 400.0


def test_errors_match_reference():
    f = fn()
    with pytest.raises(ValueError):
        predict_ttft(f, 0)
    with pytest.raises(ValueError):
        batch_delay(f, 0)
    with pytest.raises(ValueError):
        deadline_margin(f, 1, -1.0, 1)
    with pytest.raises(ValueError):
        deadline_margin(f, 1, 0.0, 0)
    with pytest.raises(ConfigError):
        fn(t0=0.0)
    with pytest.raises(ConfigError):
        fn(slo=400.0)


def test_kv_cap_and_flat_latency():
    f = fn()
    assert max_batch_size(f, free_gpu_mem_bytes=350_000_000) == 3
    flat = fn(alpha=0.0)
    assert max_batch_size(flat) == 2 ** 31
    assert max_batch_size(flat, free_gpu_mem_bytes=1_000_000_000) == 10


def test_queue_fill_expire_margin():
    f = fn()
    q = BatchQueue(f, "g0", max_batch=3)
    for i in range(3):
        q.enqueue(i, 0.0)
    d = schedule_round([q], {"g0": 0}, now=0.0)
    assert d == [FlushDecision("7b-chat", "g0", (0, 1, 2), "fill", None)]
    q.enqueue(9, 100.0)
    assert q.expire_deadline == 100.0 + batch_delay(f, 1)
    assert schedule_round([q], {"g0": 0}, now=100.0) == []
    d = schedule_round([q], {"g0": 0}, now=q.expire_deadline)
    assert d[0].reason == "expire" and d[0].request_ids == (9,)
    # margin triage: heavy contention makes a young queue flush early
    q.enqueue(10, 0.0)
    d = schedule_round([q], {"g0": 4}, now=0.0)
    assert d and d[0].reason == "margin" and d[0].margin_ms < 100.0


def _random_round(mod, rng, n_fn):
    fns, queues = [], []
    for i in range(n_fn):
        t0 = rng.uniform(100, 900)
        alpha = rng.choice([0.0, rng.uniform(10, 200)])
        slo = t0 * rng.uniform(1.5, 6)
        arts = (mod.ArtifactSpec(mod.ArtifactKind.ADAPTER_MODEL, 10, 1.0, 0.5),)
        f = mod.FunctionSpec(f"f{i}", arts, slo, t0, alpha, 1.0, rng.randint(0, 10**8), 0.0,
                             backbone_id="bb")
        fns.append(f)
    return fns


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present in this container")
def test_schedule_round_matches_reference():
    sys.path.insert(0, REF_SRC)
    try:
        from slorasim import batching as ref_b
        from slorasim import core as ref_core
    finally:
        sys.path.remove(REF_SRC)
    import paper_2505_14468_b200.spec as ours_core
    from paper_2505_14468_b200 import batching as ours_b

    for seed in range(200):
        rng = random.Random(seed)
        n_fn = rng.randint(1, 8)
        specs = {}
        for mod, key in ((ref_core, "ref"), (ours_core, "ours")):
            specs[key] = _random_round(mod, random.Random(seed * 7 + 1), n_fn)
        arrivals = [(rng.randrange(n_fn), rng.uniform(0, 3000)) for _ in range(rng.randint(0, 40))]
        arrivals.sort(key=lambda a: a[1])
        now = rng.uniform(0, 4000)
        cont = {"g0": rng.randint(0, 3), "g1": rng.randint(0, 3)}
        results = []
        for bmod, key in ((ref_b, "ref"), (ours_b, "ours")):
            fs = specs[key]
            qs = [bmod.BatchQueue(f, "g%d" % (i % 2), bmod.max_batch_size(f, 10**9))
                  for i, f in enumerate(fs)]
            for rid, (fi, t) in enumerate(arrivals):
                if t <= now:
                    qs[fi].enqueue(rid, t)
            ds = bmod.schedule_round(qs, dict(cont), now, tick_ms=10.0)
            results.append([(d.function_id, d.gpu_id, d.request_ids, d.reason,
                             None if d.margin_ms is None else round(d.margin_ms, 9)) for d in ds])
            results.append([(q.n, q.expire_deadline) for q in qs])
        assert results[0] == results[2], seed
        assert results[1] == results[3], seed
        for a, b in zip(specs["ref"], specs["ours"]):
            for bsz in (1, 2, 7):
                assert ref_b.predict_ttft(a, bsz) == ours_b.predict_ttft(b, bsz)
                assert ref_b.batch_delay(a, bsz) == ours_b.batch_delay(b, bsz)
            assert ref_b.max_batch_size(a) == ours_b.max_batch_size(b)
            assert math.isclose(ref_b.deadline_margin(a, 2, 5.0, 3), ours_b.deadline_margin(b, 2, 5.0, 3))
