"""Offload (§8 f2): the eviction policy is decision-identical to the reference's
select_evictions (CPU, where /root/reference is importable), and the memory moves are real
(GPU): an adapter demoted to the pinned container tier leaves HBM, its host copy is
byte-identical, and promoting it back restores bit-identical decode outputs."""
import os
import random
import sys

import numpy as np
import pytest
import torch

from paper_2505_14468_b200 import offload as ours
from paper_2505_14468_b200.spec import ArtifactKind

REF_SRC = "/root/reference/pkg/src"


def test_request_and_policy_basics():
    with pytest.raises(ValueError):
        ours.OffloadRequest("gpu0", 0)
    R = ours.ResidentValue
    res = [R("a", ArtifactKind.ADAPTER_MODEL, 100, 1.0), R("b", ArtifactKind.ADAPTER_MODEL, 100, 5.0)]
    ev = ours.select_evictions(ours.OffloadRequest("gpu0", 50), res, [])
    assert [(e.function_id, e.destination) for e in ev] == [("a", "discard")]
    assert ours.select_evictions(ours.OffloadRequest("gpu0", 50), res, [], free_bytes=60) == []
    with pytest.raises(ours.InsufficientEvictableMemory):
        ours.select_evictions(ours.OffloadRequest("gpu0", 150, frozenset({"b"})), res, [])
    ev = ours.select_evictions(ours.OffloadRequest("gpu0", 150), res, [], container_free={"c0": 100})
    assert [e.destination for e in ev] == ["c0", "discard"]


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present in this container")
def test_select_evictions_decision_identical_to_reference():
    sys.path.insert(0, REF_SRC)
    try:
        from slorasim import core as rc
        from slorasim import offload as ro
    finally:
        sys.path.remove(REF_SRC)
    rng = random.Random(7)
    K = rc.ArtifactKind
    n_checked = n_raised = 0
    for trial in range(400):
        fns = []
        for b in range(rng.randint(1, 3)):
            bid = f"bb{b}"
            fns.append(rc.FunctionSpec(bid, (rc.ArtifactSpec(K.BACKBONE_MODEL, 10, 1.0, 1.0),),
                                       100.0, 10.0, 1.0, 1.0, 0, 0.0))
            for a in range(rng.randint(0, 4)):
                fns.append(rc.FunctionSpec(f"{bid}-a{a}", (rc.ArtifactSpec(K.ADAPTER_MODEL, 10, 1.0, 1.0),),
                                           100.0, 10.0, 1.0, 1.0, 0, 0.0, backbone_id=bid))
        cat = rc.FunctionCatalog(fns)
        resident = []
        for f in fns:
            kinds = [K.BACKBONE_MODEL if f.backbone_id is None else K.ADAPTER_MODEL, K.KERNEL, K.LIBRARY]
            for k in kinds:
                if rng.random() < 0.75:
                    w = rng.choice([1, 5, 20, 100, 400]) * 1_000_000
                    resident.append(ro.ResidentValue(f.id, k, w, rng.choice([0.0, 0.5, 1.0, 3.0, 10.0])))
        if not resident:
            continue
        total = sum(r.weight for r in resident)
        req_bytes = rng.randint(1, max(2, int(total * 1.1)))
        protected = frozenset(f.id for f in fns if rng.random() < 0.15)
        free = rng.choice([0, 0, 1_000_000, 50_000_000])
        room = {f"c{i}": rng.choice([0, 50, 200, 1000]) * 1_000_000 for i in range(rng.randint(0, 3))}
        ctx = rng.choice([0, 473_000_000])
        args = dict(free_bytes=free, container_free=room, context_overhead_bytes=ctx)
        got = exp = None
        try:
            exp = ro.select_evictions(ro.OffloadRequest("gpu0", req_bytes, protected), resident, cat, **args)
        except ro.InsufficientEvictableMemory:
            exp = "raise"
        try:
            got = ours.select_evictions(ours.OffloadRequest("gpu0", req_bytes, protected), resident, cat, **args)
        except ours.InsufficientEvictableMemory:
            got = "raise"
        if exp == "raise":
            assert got == "raise", trial
            n_raised += 1
            continue
        assert [(e.function_id, e.kind.value, e.gpu_id, e.size_bytes, e.destination) for e in got] == \
               [(e.function_id, e.kind.value, e.gpu_id, e.size_bytes, e.destination) for e in exp], trial
        n_checked += 1
    assert n_checked > 100 and n_raised > 10


@pytest.mark.gpu
def test_adapter_demotion_and_promotion_are_real_moves(golden):
    from paper_2505_14468_b200.config import TINY, TINY_LORA, init_adapter, init_backbone
    from paper_2505_14468_b200.model import MultiLoraModel
    from paper_2505_14468_b200.preload import HostArtifactStore, Preloader

    seed = int(golden["seed"])
    m = MultiLoraModel(TINY, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=4, max_rank=16,
                       max_tokens=256)
    m.load_backbone(init_backbone(TINY, seed))
    for a in range(3):
        m.pool.load(a, init_adapter(TINY, TINY_LORA, seed, a), TINY_LORA)
    prompts, ids = [[5, 9, 200, 31], [7, 7, 7], [100, 2, 3]], [0, 1, 2]

    def run():
        seqs, logits = m.prefill(prompts, ids)
        out = logits.float().cpu().numpy()
        for s in seqs:
            m.free_seq(s)
        return out

    before = run()
    blob1 = m.pool.blobs[1].clone()
    led0 = m.memory_ledger()
    store = HostArtifactStore(8 << 20)
    off = ours.Offloader(m, store, {"f0": 0, "f1": 1, "f2": 2}, backbone_fid="tiny")
    ev = [ours.Eviction("f1", ArtifactKind.ADAPTER_MODEL, "gpu0", blob1.numel() * 2, "host0a"),
          ours.Eviction("f2", ArtifactKind.ADAPTER_MODEL, "gpu0", blob1.numel() * 2, "discard")]
    done = off.apply(ev)
    assert done[0][0] > 0.0 and done[1][0] == 0.0
    assert m.pool.blobs[1] is None and m.pool.blobs[2] is None
    led1 = m.memory_ledger()
    assert led0["adapter_pool"] - led1["adapter_pool"] == 2 * blob1.numel() * 2
    host = torch.from_numpy(store.view("offload/f1").copy()).view(torch.bfloat16)
    assert torch.equal(host, blob1.cpu())
    with pytest.raises(ours.StaleStateError):
        off.apply(ev[:1])
    pre = Preloader(store, m.device)
    off.promote("f1", pre)
    m.pool.load(2, init_adapter(TINY, TINY_LORA, seed, 2), TINY_LORA)
    after = run()
    np.testing.assert_array_equal(after, before)
    store.close()
