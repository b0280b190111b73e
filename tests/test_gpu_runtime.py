"""GPU: the serving runtime (batcher -> merged prefill -> merged decode), the artifact
pre-loader and the calibration bridge, end to end on the tiny config."""

import numpy as np
import pytest
import torch

from paper_2505_14468_b200.batching import max_batch_size, predict_ttft
from paper_2505_14468_b200.calibrate import profile_function_spec
from paper_2505_14468_b200.config import TINY, TINY_LORA, init_adapter, init_backbone
from paper_2505_14468_b200.model import MultiLoraModel
from paper_2505_14468_b200.preload import HostArtifactStore, NcclComm, Preloader
from paper_2505_14468_b200.runtime import ServingRuntime
from paper_2505_14468_b200.spec import ArtifactKind, ArtifactSpec, FunctionSpec

pytestmark = pytest.mark.gpu


def _model(golden, dtype=torch.float32, max_seqs=16, n_slots=8):
    seed = int(golden["seed"])
    w = init_backbone(TINY, seed)
    ads = [init_adapter(TINY, TINY_LORA, seed, a) for a in range(4)]
    m = MultiLoraModel(TINY, dtype=dtype, max_seqs=max_seqs, max_ctx=128, n_slots=n_slots,
                       max_rank=16, max_tokens=2048)
    m.load_backbone(w)
    return m, w, ads


def _prompts(golden):
    ip = golden["prompt_indptr"]
    return [list(map(int, golden["prompt_flat"][ip[i]:ip[i + 1]])) for i in range(len(ip) - 1)]


def _spec(fid, t0=5.0, alpha=1.0):
    arts = (ArtifactSpec(ArtifactKind.ADAPTER_MODEL, 10, 1.0, 1.0),)
    return FunctionSpec(fid, arts, 5 * t0, t0, alpha, 1.0, 0, 0.0, backbone_id="tiny")


def test_preloader_h2d_then_runtime_serves_golden_tokens(golden):
    """Adapters enter HBM through the pinned-host pre-loader; four LoRA functions are served
    through batcher rounds as merged mixed-adapter prefill/decode; fp32 greedy tokens are
    bit-exact with the transformers golden."""
    m, w, ads = _model(golden)
    store = HostArtifactStore(64 << 20)
    pre = Preloader(store, m.device, chunk_bytes=1 << 20)
    for a, ad in enumerate(ads):
        store.put(f"adapter{a}", m.pool.pack(ad, TINY_LORA.rank))
    for a in range(4):
        dev, ev = pre.load(f"adapter{a}")
        ev.synchronize()
        m.pool.install(a, dev.view(torch.bfloat16), TINY_LORA)
    assert pre.timed_load_ms("adapter0") > 0
    funcs = {f"fn{a}": (_spec(f"fn{a}"), a) for a in range(4)}
    rt = ServingRuntime(m, funcs)
    prompts = _prompts(golden)
    ids = list(map(int, golden["adapter_ids"]))
    n_new = int(golden["n_new"])
    for i, (p, a) in enumerate(zip(prompts, ids)):
        rt.submit(i, f"fn{a}", p, n_new)
    done = rt.run_until_idle()
    assert len(done) == len(prompts)
    toks = np.stack([np.asarray(sorted(done, key=lambda r: r.request_id)[i].generated[:n_new])
                     for i in range(len(prompts))])
    assert np.array_equal(toks, golden["tokens"])
    assert all(r.first_token_ms is not None and r.done_ms >= r.first_token_ms for r in done)
    store.close()


def test_mixed_rounds_serve_golden_tokens(golden):
    """Staggered arrivals, so rounds have new prompts AND running sequences: with mixed rounds
    the running sequences' tokens ride in the round's prefill forward (1-token segments with a
    cached prefix); fp32 greedy tokens stay bit-exact with the transformers golden, and equal
    the separate prefill + decode rounds'."""
    out = {}
    for mixed in (True, False):
        m, w, ads = _model(golden)
        for a, ad in enumerate(ads):
            m.pool.load(a, ad, TINY_LORA)
        funcs = {f"fn{a}": (_spec(f"fn{a}"), a) for a in range(4)}
        # a tick far beyond every deadline margin: each queue flushes at the next round
        rt = ServingRuntime(m, funcs, tick_ms=1e6, mixed_rounds=mixed)
        prompts = _prompts(golden)
        ids = list(map(int, golden["adapter_ids"]))
        n_new = int(golden["n_new"])
        half = len(prompts) // 2
        for i in range(half):
            rt.submit(i, f"fn{ids[i]}", prompts[i], n_new)
        for _ in range(200):       # the first half is running before the rest arrives
            rt.step()
            if rt.active:
                break
        for k in range(3):
            rt.step()
        for i in range(half, len(prompts)):
            rt.submit(i, f"fn{ids[i]}", prompts[i], n_new)
        done = rt.run_until_idle()
        assert len(done) == len(prompts)
        toks = np.stack([np.asarray(sorted(done, key=lambda r: r.request_id)[i].generated[:n_new])
                         for i in range(len(prompts))])
        assert np.array_equal(toks, golden["tokens"])
        out[mixed] = (toks, rt.mixed_steps)
    assert out[True][1] > 0 and out[False][1] == 0
    assert np.array_equal(out[True][0], out[False][0])


def test_nccl_broadcast_world1_roundtrip():
    """The pre-loader's own NCCL communicator (world 1 on the single-GPU box): one host read,
    pipelined H2D + broadcast, bytes land intact."""
    store = HostArtifactStore(8 << 20)
    data = np.random.default_rng(0).integers(0, 255, size=5_000_000, dtype=np.uint8)
    store.put("blob", data)
    pre = Preloader(store, torch.device("cuda", 0), chunk_bytes=1 << 20)
    comm = NcclComm(0, 1)
    out = pre.load_broadcast("blob", 0, comm)
    pre.wait()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), data)
    comm.close()
    store.close()


def test_calibration_feeds_the_batcher(golden):
    m, w, ads = _model(golden, dtype=torch.bfloat16)
    m.pool.load(0, ads[0], TINY_LORA)
    spec, raw = profile_function_spec(m, "tiny-chat", 0, backbone_id="tiny", prompt_len=24,
                                      max_new_tokens=8, batch_sizes=(1, 2, 4, 8))
    assert spec.prefill_base_ms > 0 and spec.prefill_marginal_ms >= 0
    assert spec.decode_ms_per_token > 0
    # the pool reserves max_ctx positions per sequence slot (memory_ledger's kv_slot_bytes)
    assert spec.kv_cache_bytes_per_request == m.memory_ledger()["kv_slot_bytes"]
    assert spec.slo_ttft_ms == pytest.approx(5 * spec.prefill_base_ms)
    assert predict_ttft(spec, 1) == spec.prefill_base_ms
    assert max_batch_size(spec) >= 1
    assert len(raw["prefill_ms"]) == 4


_LEDGER_CHECK = """
import sys, numpy as np, torch
from paper_2505_14468_b200.config import TINY, TINY_LORA, init_adapter, init_backbone
from paper_2505_14468_b200.model import MultiLoraModel
dtype = getattr(torch, sys.argv[1]); seed = int(sys.argv[2])
def requested():
    return torch.cuda.memory_stats()["requested_bytes.all.current"]
torch.cuda.init(); torch.cuda.synchronize(); base = requested()
m = MultiLoraModel(TINY, dtype=dtype, max_seqs=8, max_ctx=128, n_slots=8, max_rank=16, max_tokens=512)
m.load_backbone(init_backbone(TINY, seed))
for a in range(3):
    m.pool.load(a, init_adapter(TINY, TINY_LORA, seed, a), TINY_LORA)
torch.cuda.synchronize()
led = m.memory_ledger()
assert led["total"] == requested() - base, (led, requested() - base)
assert led["kv_pool"] == m.max_seqs * led["kv_slot_bytes"]
assert led["backbone"] >= m.backbone_bytes()
one = led["adapter_pool"] // 3
assert one == m.pool.resident_bytes() // 3 and one > 0
assert (led["adapter_stacked_rows"] > 0) == (dtype == torch.bfloat16)
m.pool.evict(2)
torch.cuda.synchronize()
led2 = m.memory_ledger()
assert led["adapter_pool"] - led2["adapter_pool"] == one
assert led2["total"] == requested() - base, (led2, requested() - base)
print("ledger ok", led)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_memory_ledger_matches_allocator(golden, dtype):
    """§8 a7: the ledger categories (backbone / adapter residents / KV pool / workspaces) add up
    to exactly the bytes the caching allocator handed out for the model, and evicting an
    adapter moves both by the adapter's bytes (the reference books one backbone per GPU plus
    one reservation per resident adapter, ledger.py:108-134).  Runs in a fresh process so no
    other test's tensors are allocated or freed inside the measured window."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _LEDGER_CHECK, dtype, str(int(golden["seed"]))],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ledger ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_runtime_admission_cold_loads_and_offload_keep_golden_tokens(golden):
    """Dispatch admission (reference _try_dispatch, engine.py:711-853) with a pool of TWO adapter
    slots for four functions whose adapters live in the pinned container tier: missing
    adapters are loaded at dispatch through the pre-loader (cold start), idle ones are demoted
    by select_evictions + Offloader (D2H) to make room, KV-short flushes are deferred; the
    fp32 greedy tokens stay bit-exact with the transformers golden."""
    from paper_2505_14468_b200.offload import Offloader
    m, w, ads = _model(golden, max_seqs=6, n_slots=2)   # 6 KV slots for 16 requests: deferrals
    store = HostArtifactStore(64 << 20)
    pre = Preloader(store, m.device, chunk_bytes=1 << 20)
    for a, ad in enumerate(ads):
        store.put(f"adapter{a}", m.pool.pack(ad, TINY_LORA.rank))
    funcs = {f"fn{a}": (_spec(f"fn{a}"), -1) for a in range(4)}
    adapters = {f"fn{a}": (f"adapter{a}", TINY_LORA) for a in range(4)}
    off = Offloader(m, store, {})
    rt = ServingRuntime(m, funcs, store=store, adapters=adapters, preloader=pre, offloader=off)
    prompts = _prompts(golden)
    ids = list(map(int, golden["adapter_ids"]))
    n_new = int(golden["n_new"])
    for i, (p, a) in enumerate(zip(prompts, ids)):
        rt.submit(i, f"fn{a}", p, n_new)
    with pytest.raises(ValueError):
        rt.submit(99, "fn0", [1] * 120, 10)   # prompt + new tokens > max_ctx: rejected
    done = rt.run_until_idle()
    assert len(done) == len(prompts)
    toks = np.stack([np.asarray(sorted(done, key=lambda r: r.request_id)[i].generated[:n_new])
                     for i in range(len(prompts))])
    assert np.array_equal(toks, golden["tokens"])
    assert any(v for v in rt.cold_ms.values())      # some requests waited for a cold load
    assert off.demoted or len({f for f, (_, s) in rt.functions.items() if s >= 0}) <= 2
    assert len(m.free_seqs) == 6                      # every KV slot returned
    store.close()


def test_runtime_graph_decode_buckets_bf16(golden):
    """bf16 serving with the captured decode graphs (batch-size buckets, padded rows on the
    reserved scratch sequence): greedy tokens agree with the golden up to each request's first
    position whose oracle margin is below TAU, and every decode step ran from a graph."""
    m, w, ads = _model(golden, dtype=torch.bfloat16, max_seqs=17)
    for a, ad in enumerate(ads):
        m.pool.load(a, ad, TINY_LORA)
    funcs = {f"fn{a}": (_spec(f"fn{a}"), a) for a in range(4)}
    rt = ServingRuntime(m, funcs)
    assert rt.graphs is not None
    prompts = _prompts(golden)
    ids = list(map(int, golden["adapter_ids"]))
    n_new = int(golden["n_new"])
    for i, (p, a) in enumerate(zip(prompts, ids)):
        rt.submit(i, f"fn{a}", p, n_new)
    done = sorted(rt.run_until_idle(), key=lambda r: r.request_id)
    assert rt.graph_steps == rt.decode_steps > 0
    gold, margin = golden["tokens"], golden["margin"]
    for r in range(gold.shape[0]):
        for s in range(gold.shape[1]):
            assert done[r].generated[s] == gold[r, s] or margin[r, s] < 0.05
            if margin[r, s] < 0.05:
                break
    rep = rt.report()
    assert rep["requests"] == len(prompts) and rep["ttft_ms"]["p50"] > 0


def test_calibration_on_the_flash_prefill_path():
    """profile_function_spec at head_dim 128 (the tcgen05 flash prefill + stacked small-batch
    LoRA path of the 7B/13B calibration, tools/calibrate_b200.py): forward() called with
    segments and no host slots must plan without them (regression: the plan cache keyed on
    host slots the non-SGMV path does not have)."""
    from paper_2505_14468_b200.config import BackboneConfig, LoraConfig
    cfg = BackboneConfig("small128", hidden=512, layers=2, heads=4, kv_heads=4, head_dim=128,
                         ffn=1024, vocab=1000)
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=8, max_ctx=64, n_slots=2, max_rank=16,
                       max_tokens=8 * 32)
    m.random_backbone(seed=0)
    m.pool.load_random(0, LoraConfig(16, 32.0, ("q", "k", "v", "o")), seed=1)
    spec, raw = profile_function_spec(m, "small-chat", 0, backbone_id="small128", prompt_len=24,
                                      max_new_tokens=8, batch_sizes=(1, 2, 4))
    assert spec.prefill_base_ms > 0 and spec.decode_ms_per_token > 0
    assert len(raw["prefill_ms"]) == 3
