"""Wire formats (§8 f4): the trace CSV and request CSV are interchangeable with the
reference's own reader/writer (CPU, where /root/reference is importable), and a trace replays
through the serving runtime end to end (GPU)."""
import csv
import math
import os
import sys

import pytest

from paper_2505_14468_b200 import wire
from paper_2505_14468_b200.spec import ConfigError

REF_SRC = "/root/reference/pkg/src"


def _ref():
    sys.path.insert(0, REF_SRC)
    try:
        from slorasim import engine, metrics, workload
    finally:
        sys.path.remove(REF_SRC)
    return engine, metrics, workload


def test_trace_roundtrip_and_errors(tmp_path):
    recs = [wire.TraceRecord("b", 10.5, 60, 64), wire.TraceRecord("a", 10.5, 12, 3),
            wire.TraceRecord("a", 0.0, 7, 1)]
    p = tmp_path / "t.csv"
    wire.write_trace_csv(recs, p)
    got = wire.read_trace_csv(p)
    assert got == sorted(recs, key=lambda r: (r.arrival_ms, r.function_id))
    bad = tmp_path / "bad.csv"
    bad.write_text("function_id,arrival_ms\nx,1\n")
    with pytest.raises(ConfigError):
        wire.read_trace_csv(bad)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present in this container")
def test_formats_interchangeable_with_reference(tmp_path):
    engine, metrics, workload = _ref()
    tr = workload.generate_trace(workload.CovClass.BURSTY, 30.0, 1.0, 3, function_id="7b-chat")
    p = tmp_path / "ref.csv"
    workload.write_trace_csv(tr, p)
    ours = wire.read_trace_csv(p)
    assert [(r.function_id, r.arrival_ms, r.prompt_tokens, r.output_tokens) for r in ours] == \
           [(r.function_id, r.arrival_ms, r.prompt_tokens, r.output_tokens) for r in tr]
    q = tmp_path / "ours.csv"
    wire.write_trace_csv(ours, q)
    assert q.read_text() == p.read_text()
    assert wire.REQUEST_CSV_COLUMNS == metrics.REQUEST_CSV_COLUMNS

    # one finished request, written by both writers
    class R:   # runtime request shape (segments.Request)
        request_id, function_id, arrival_ms = 7, "7b-chat", 12.25
        first_token_ms, done_ms, generated = 40.5, 140.5, [1] * 11
    rec = engine.RequestRecord(7, "7b-chat", 12.25, 60, 11, dispatch_ms=13.0, first_token_ms=40.5,
                               completion_ms=140.5, batch_size=1)
    rec.cold_start_breakdown["backbone_load"] = 3.5
    metrics.write_requests_csv([rec], tmp_path / "ref_req.csv")
    wire.write_requests_csv([R()], tmp_path / "our_req.csv", cold={7: {"backbone_load": 3.5}})
    assert (tmp_path / "our_req.csv").read_text() == (tmp_path / "ref_req.csv").read_text()
    R.generated = [1]
    row = wire.request_row(R())
    assert math.isnan(float(row[4]))


@pytest.mark.gpu
def test_trace_replays_through_runtime(golden, tmp_path):
    import torch
    from paper_2505_14468_b200.config import TINY, TINY_LORA, init_adapter, init_backbone
    from paper_2505_14468_b200.model import MultiLoraModel
    from paper_2505_14468_b200.runtime import ServingRuntime
    from paper_2505_14468_b200.spec import ArtifactKind, ArtifactSpec, FunctionSpec

    seed = int(golden["seed"])
    m = MultiLoraModel(TINY, dtype=torch.bfloat16, max_seqs=16, max_ctx=128, n_slots=4,
                       max_rank=16, max_tokens=2048)
    m.load_backbone(init_backbone(TINY, seed))
    fns = {}
    for a in range(3):
        m.pool.load(a, init_adapter(TINY, TINY_LORA, seed, a), TINY_LORA)
        arts = (ArtifactSpec(ArtifactKind.ADAPTER_MODEL, 10, 1.0, 1.0),)
        fns[f"f{a}"] = (FunctionSpec(f"f{a}", arts, 50.0, 5.0, 1.0, 1.0, 0, 0.0, backbone_id="tiny"), a)
    rt = ServingRuntime(m, fns)
    recs = [wire.TraceRecord(f"f{i % 3}", 4.0 * i, 5 + i, 1 + i % 4) for i in range(12)]
    p = tmp_path / "trace.csv"
    wire.write_trace_csv(recs, p)
    done = wire.replay(rt, wire.read_trace_csv(p), TINY.vocab, seed=1, max_ctx=128)
    assert len(done) == 12
    by_id = {r.request_id: r for r in done}
    for i, rec in enumerate(sorted(recs, key=lambda r: (r.arrival_ms, r.function_id))):
        r = by_id[i]
        assert r.function_id == rec.function_id and len(r.generated) == rec.output_tokens
        assert r.first_token_ms >= r.arrival_ms and r.done_ms >= r.first_token_ms
    out = tmp_path / "requests.csv"
    wire.write_requests_csv(done, out)
    rows = list(csv.reader(open(out)))
    assert rows[0] == wire.REQUEST_CSV_COLUMNS and len(rows) == 13
