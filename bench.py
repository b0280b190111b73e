"""Benchmark: multi-LoRA decode tokens/s on the Llama-2-7B shape (BASELINE.json config 2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload config2|config3] [--ctx C] [--no-cpu-baseline] [--no-prefill]

config2 (default, the `metric` line): a step is one mixed-adapter decode step of 64 sequences
per GPU (32 rank-16 adapters on q,k,v,o, per-token adapter ids uniform with seed 0) at
context 128 over the full 32-layer 7B-shape bf16 backbone (random init, synthetic tokens),
lm_head and greedy argmax included, replayed as one CUDA graph.  The line also carries a
`prefill_config3` summary (BASELINE config 3: 13B shape, 128 adapters of rank {8,16,64},
8 x 2048-token prefill on one GPU).

config3 (--workload config3): the 13B prefill as the line's workload (prefill tokens/s,
tensor-pipe roofline of the backbone GEMMs).

Data parallel: every GPU holds a backbone replica; a global synthetic request
stream of 64 x N requests is split across the ranks by dp.route (join-shortest-queue), each
rank decodes its share, no collective in the step.  `--gpus N` outside torchrun re-launches
itself under torch.distributed.run (one process per GPU, NCCL); N > visible GPUs fails.
Timing: CUDA events on the launching stream, barrier + synchronize on both sides, max over
ranks.  The 13.5 GB of weights streamed every step exceed the 126 MB L2 (no flush needed).

--impl reference times the oracle port (oracle/llama_lora.py, numpy fp32 on all host
cores) on a bounded sample of the same workload — the reference (slorasim) is a simulator
with no forward of its own; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "tokens/s"
BATCH, N_ADAPTERS, RANK, ALPHA = 64, 32, 16, 32.0
P3, L3, N_AD3 = 8, 2048, 128          # config 3: prompts x tokens, adapters (ranks {8,16,64})


def metric_name(workload: str, ctx: int) -> str:
    if workload == "config3":
        return ("multi-LoRA prefill tokens/s (Llama-2-13B shape, 128 adapters r{8,16,64}, "
                "8 x 2048-token prompts)")
    return f"multi-LoRA decode tokens/s (Llama-2-7B shape, 32 x r16 adapters, batch 64, ctx {ctx})"


def config_dict(workload: str, ctx: int, world: int) -> dict:
    """The workload description — identical in both arms (same keys, same values)."""
    if workload == "config3":
        return {"workload": "config3: llama2-13b-shape bf16 prefill, 8 x 2048-token prompts, "
                            "128 adapters of rank {8,16,64} on q,k,v,o",
                "prompts_per_gpu": P3, "prompt_tokens": L3, "global_batch": P3 * world,
                "adapters": N_AD3, "ranks": "8/16/64 (seeded)", "lora_targets": "q,k,v,o",
                "parallelism": f"dp{world} (replicas)", "l2": "inputs > L2 (26 GB weights)"}
    return {"workload": f"config2: llama2-7b-shape bf16 decode, 32 x r16 LoRA (q,k,v,o), batch 64, "
                        f"ctx {ctx}",
            "batch_per_gpu": BATCH, "global_batch": BATCH * world, "ctx": ctx,
            "adapters": N_ADAPTERS, "rank": RANK, "lora_targets": "q,k,v,o",
            "parallelism": f"dp{world} (replicas)",
            "l2": "inputs > L2: 13.5 GB weights + 4.3 GB KV streamed per step"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def global_stream(world: int, seed: int = 0):
    """The synthetic request stream of a data-parallel step: BATCH requests per GPU, each
    (request id, prompt, max_new_tokens, adapter id); adapters uniform (seed 0)."""
    rng = np.random.default_rng(seed)
    n = BATCH * world
    ads = rng.integers(0, N_ADAPTERS, size=n)
    return [(i, [1] * 128, 32, int(ads[i])) for i in range(n)]


def my_slots(rank: int, world: int) -> np.ndarray:
    from paper_2505_14468_b200 import dp
    mine = dp.shard(global_stream(world), rank, world)
    assert len(mine) == BATCH, "equal-cost requests: join-shortest-queue deals BATCH per rank"
    return np.array([r[3] for r in mine], dtype=np.int32)


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        p = {}
    hbm = float(p.get("hbm_gbs", 6650.0))
    tf = float(p.get("bf16_tflops_sustained", 1380.0))
    src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in p else "fallback (B200_PROFILING.md)"
    return hbm, tf, src


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------ CPU oracle
def _oracle_layer_model(cfg_full, n_adapters, ranks, n_seqs, ctx, seed=0, max_pos=None):
    """One decoder layer of ``cfg_full`` in the numpy fp32 oracle with ``n_adapters`` adapters
    (ranks[a]) on q,k,v,o and ``n_seqs`` sequences of ``ctx`` cached positions."""
    from oracle.llama_lora import OracleModel
    from paper_2505_14468_b200.config import BackboneConfig

    cfg1 = BackboneConfig("one-layer", cfg_full.hidden, 1, cfg_full.heads, cfg_full.kv_heads,
                          cfg_full.head_dim, cfg_full.ffn, cfg_full.vocab)
    rng = np.random.default_rng(seed)
    f32 = np.float32

    def rn(*shape, s=0.02):
        return rng.standard_normal(shape, dtype=f32) * f32(s)

    d = cfg1.hidden
    w = {"embed": rn(cfg1.vocab, d, s=1.0), "final_norm": np.ones(d, f32),
         "lm_head": rn(cfg1.vocab, d), "layers.0.input_norm": np.ones(d, f32),
         "layers.0.post_norm": np.ones(d, f32), "layers.0.wq": rn(d, d),
         "layers.0.wk": rn(d, d), "layers.0.wv": rn(d, d), "layers.0.wo": rn(d, d),
         "layers.0.w_gate": rn(cfg1.ffn, d), "layers.0.w_up": rn(cfg1.ffn, d),
         "layers.0.w_down": rn(d, cfg1.ffn)}
    ads = []
    for a in range(n_adapters):
        ad = {}
        for t in ("q", "k", "v", "o"):
            ad[f"layers.0.{t}.A"] = rn(int(ranks[a]), d, s=1 / np.sqrt(d))
            ad[f"layers.0.{t}.B"] = rn(d, int(ranks[a]))
        ads.append(ad)
    m = OracleModel(cfg1, w, ads, [2.0] * n_adapters, ("q", "k", "v", "o"),
                    max_pos=max_pos or ctx + 8)
    for _ in range(n_seqs):
        m.kv.append([(rn(ctx, cfg1.kv_heads, cfg1.head_dim, s=1.0),
                      rn(ctx, cfg1.kv_heads, cfg1.head_dim, s=1.0))])
    return m, rng


class CpuOracleSample:
    """A bounded sample of the workload in the numpy fp32 oracle on all host cores.
    config2: one 7B decoder layer at batch 64 / ctx 128 (+ lm_head); a step = layer x 32.
    config3: one 13B decoder layer over ONE 2048-token prompt (+ lm_head of its last token);
    a step = (layer x 40 + lm_head) x 8 prompts."""

    def __init__(self, workload: str, ctx: int = 128):
        from paper_2505_14468_b200.config import LLAMA2_7B, LLAMA2_13B

        self.workload = workload
        self.cores = len(os.sched_getaffinity(0))
        if workload == "config3":
            self.full = LLAMA2_13B
            ranks = np.random.default_rng(0).choice([8, 16, 64], size=N_AD3)
            self.m, rng = _oracle_layer_model(self.full, 4, ranks[:4], 0, 0, max_pos=L3 + 8)
            self.toks = rng.integers(1, self.full.vocab, size=L3)
            self.units = P3 * L3
            self.sample = (f"numpy fp32 oracle on {self.cores} host threads ({cpu_model()}): 1 of 40 "
                           f"13B decoder layers over 1 of 8 prompts (2048 tokens, rank-{int(ranks[0])}"
                           f" adapter) + lm_head; step = (layer x 40 + lm_head) x 8 prompts")
        else:
            self.full = LLAMA2_7B
            self.m, rng = _oracle_layer_model(self.full, N_ADAPTERS, [RANK] * N_ADAPTERS, BATCH, ctx)
            self.ctx = ctx
            self.slots = my_slots(0, 1)
            self.toks = rng.integers(1, self.full.vocab, size=BATCH)
            self.units = BATCH
            self.sample = (f"numpy fp32 oracle on {self.cores} host threads ({cpu_model()}): 1 of 32 "
                           f"7B decoder layers (batch {BATCH}, ctx {ctx}, {N_ADAPTERS} r{RANK} "
                           f"adapters on q,k,v,o) + lm_head per step; layer time x32 extrapolated")

    def step_seconds(self) -> float:
        m = self.m
        if self.workload == "config3":
            m.kv = []
            m.kv.append([(np.zeros((0, self.full.kv_heads, self.full.head_dim), np.float32),) * 2])
            t0 = time.perf_counter()
            h = m._forward(self.toks, np.arange(L3), np.array([0, L3]), np.array([0]), [0])
            t1 = time.perf_counter()
            m.logits(h[-1:])
            t2 = time.perf_counter()
            return P3 * (self.full.layers * (t1 - t0) + (t2 - t1))
        for s in range(BATCH):  # rewind to the context (constant attended length)
            kc, vc = m.kv[s][0]
            m.kv[s][0] = (kc[:self.ctx], vc[:self.ctx])
        t0 = time.perf_counter()
        h = m._forward(self.toks, np.full(BATCH, self.ctx), np.arange(BATCH + 1), self.slots,
                       list(range(BATCH)))
        t1 = time.perf_counter()
        m.logits(h)
        t2 = time.perf_counter()
        return self.full.layers * (t1 - t0) + (t2 - t1)


def cpu_baseline_line(workload: str, ctx: int, min_seconds=10.0):
    smp = CpuOracleSample(workload, ctx)
    smp.step_seconds()
    times, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < min_seconds or len(times) < 3:
        times.append(smp.step_seconds())
    v = smp.units / statistics.median(times)
    return {"value": v, "unit": UNIT, "cores": smp.cores, "kind": "port", "cpu": cpu_model(),
            "sample": smp.sample + f", median of {len(times)} steps"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    smp = CpuOracleSample(args.workload, args.ctx)
    for _ in range(args.warmup):
        smp.step_seconds()
    t0 = time.perf_counter()
    times = [smp.step_seconds() for _ in range(args.steps)]
    elapsed = time.perf_counter() - t0
    value = smp.units * len(times) / sum(times)
    # A step is a bounded sample of the workload (the contract's reference arm): ms_per_step is
    # the measured wall time of one sample step, so steps x ms_per_step matches the run's clock;
    # value is the full workload's rate from the sample (full_step_ms_extrapolated).
    line = {"impl": "reference", "metric": metric_name(args.workload, args.ctx), "value": value,
            "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 * elapsed / max(1, len(times)), 3),
            "full_step_ms_extrapolated": round(1000.0 * smp.units / value, 3),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random init, seed 0)",
            "config": config_dict(args.workload, args.ctx, 1),
            "host_wall_s": round(elapsed, 2),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": smp.cores, "kind": "port",
                             "cpu": cpu_model(), "sample": smp.sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ ours: decode
def decode_bytes(cfg, slots, ctx):
    """Per-step algorithmic bytes by kernel class (SURVEY.md §8d definitions)."""
    B, d, qd, kvd, f = BATCH, cfg.hidden, cfg.q_dim, cfg.kv_dim, cfg.ffn
    gemm = 0
    for (N, K, n_out, res) in [(qd + 2 * kvd, d, qd + 2 * kvd, 0), (d, qd, d, 1),
                               (2 * f, d, f, 0), (d, f, d, 1)]:
        gemm += N * K * 2 + B * K * 2 + B * n_out * 2 + res * B * n_out * 2
    gemm *= cfg.layers
    gemm += cfg.vocab * d * 2 + B * d * 2 + B * cfg.vocab * 4      # lm_head (fp32 logits)
    distinct = len(set(slots.tolist()))
    lora = 0
    for t, (di, do) in {"q": (d, qd), "k": (d, kvd), "v": (d, kvd), "o": (qd, d)}.items():
        lora += distinct * RANK * (di + do) * 2 + B * di * 2 + 2 * B * do * 2
    lora *= cfg.layers
    # what the fused implementation actually moves: every slot's stacked A rows (streamed by the
    # projection GEMMs), the distinct adapters' B rows (fused expands), the fp32 v side output
    moved = cfg.layers * (4 * N_ADAPTERS * RANK * d * 2 + distinct * RANK * (qd + 2 * kvd + d) * 2
                          + 2 * B * 4 * N_ADAPTERS * RANK * 4)
    attn = cfg.layers * (B * (ctx + 1) * 2 * kvd * 2 + B * (qd + 2 * kvd) * 2 + B * qd * 2)
    return {"gemm": gemm, "lora": lora, "lora_moved": moved, "attention": attn}, distinct


def run_decode(args, rank, local_rank, world, dist):
    import torch

    from paper_2505_14468_b200 import ops, profiling
    from paper_2505_14468_b200._lib import EPI_SILU_MUL, load
    from paper_2505_14468_b200.config import LLAMA2_7B, LoraConfig
    from paper_2505_14468_b200.engine import DecodeGraph
    from paper_2505_14468_b200.model import MultiLoraModel

    CTX = args.ctx
    cfg = LLAMA2_7B
    lora = LoraConfig(RANK, ALPHA, ("q", "k", "v", "o"))
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=BATCH, max_ctx=CTX + 1,
                       n_slots=N_ADAPTERS, max_rank=RANK, max_tokens=BATCH)
    m.random_backbone(seed=0)   # every replica holds the same backbone
    for a in range(N_ADAPTERS):
        m.pool.load_random(a, lora, seed=1000 + a)
    g = torch.Generator(device=m.device).manual_seed(7 + rank)
    for l in range(cfg.layers):   # context of CTX resident tokens per sequence
        m.k_cache[l].normal_(generator=g)
        m.v_cache[l].normal_(generator=g)
    seqs = [m.alloc_seq() for _ in range(BATCH)]
    led = m.memory_ledger()   # what the reference's ResidencyLedger books per GPU
    hbm_ledger = {k: round(led[k] / 1e9, 4) for k in ("backbone", "adapter_pool",
                                                       "adapter_stacked_rows", "kv_pool",
                                                       "workspace", "total")}
    hbm_ledger["kv_slot_mb"] = round(led["kv_slot_bytes"] / 1e6, 3)
    slots = my_slots(rank, world)
    dg = DecodeGraph(m, seqs, slots.tolist(), fixed_pos=CTX)
    dg.tok.copy_(torch.randint(1, cfg.vocab, (BATCH,), generator=g, device=m.device, dtype=torch.int32))
    dg.capture()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=m.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up + timed device loop (tokens fed back on device)
    for _ in range(args.warmup):
        dg.replay()
        dg.feed_back()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            dg.replay()
            dg.feed_back()
        ev1.record(stream)
        barrier()
    my_ms = ev0.elapsed_time(ev1)
    t_ms = max_over_ranks(my_ms)
    value = world * BATCH * args.steps / (t_ms / 1000.0)
    per_rank = [BATCH * args.steps / (my_ms / 1000.0)]
    if world > 1:
        from paper_2505_14468_b200 import dp
        per_rank = [x[0] for x in dp.gather_metrics(per_rank, world)]
    launches = dg.kernels_per_step * args.steps

    # ---- end to end through host buffers (H2D inputs, D2H sampled tokens every step)
    h_tok = np.random.default_rng(1).integers(1, cfg.vocab, size=BATCH).astype(np.int32)
    for _ in range(2):
        h_tok = dg.step_host(h_tok, slots).copy()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        h_tok = dg.step_host(h_tok, slots).copy()
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = world * BATCH * args.steps / (e2e_ms / 1000.0)

    hbm_peak, tf_peak, peak_src = peaks()
    abytes, distinct = decode_bytes(cfg, slots, CTX)
    # ---- in-graph timeline: every GEMM's exit-to-exit share of the replayed step
    tl = profiling.trace_graph(lambda: DecodeGraph(m, seqs, slots.tolist(), fixed_pos=CTX))
    e2x = profiling.exit_to_exit(tl)
    gemm_n, gemm_us = e2x.get("gemm", (0, 0.0))
    span = profiling.step_span_us(tl)
    # the first traced launch (layer 0's q/k/v GEMM follows the untraced plain RMSNorm) has no
    # exit-to-exit span: scale its bytes out
    gemm_bytes_traced = abytes["gemm"] * gemm_n / (4 * cfg.layers + 1)
    gemm_gbs = gemm_bytes_traced / (gemm_us * 1e-6) / 1e9 if gemm_us else 0.0
    in_graph = {k: {"launches": n, "us_per_step": round(us, 1), "share_of_span": round(us / span, 4)}
                for k, (n, us) in e2x.items()}

    # ---- LoRA cost in the graph: the same step on the bare backbone (same weights, no LoRA
    # targets: no stacked shrink rows, no fused deltas)
    m0 = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=BATCH, max_ctx=CTX + 1,
                        n_slots=N_ADAPTERS, max_rank=RANK, max_tokens=BATCH, lora_targets=())
    m0.random_backbone(seed=0)
    m0.k_cache, m0.v_cache = m.k_cache, m.v_cache
    for _ in seqs:
        m0.alloc_seq()
    dg0 = DecodeGraph(m0, seqs, [-1] * BATCH, fixed_pos=CTX)
    dg0.tok.copy_(dg.tok)
    dg0.capture()
    for _ in range(args.warmup):
        dg0.replay()
    barrier()
    z0, z1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    z0.record(stream)
    for _ in range(args.steps):
        dg0.replay()
    z1.record(stream)
    barrier()
    t_nolora_ms = max_over_ranks(z0.elapsed_time(z1))
    del dg0, m0
    torch.cuda.empty_cache()

    # ---- the dominant kernel chained: one CUDA graph of the 32 layers' gate/up (and q/k/v)
    # GEMM launches back to back (PDL between them, every launch streaming its own layer's
    # weights, > L2), CUDA events around R replays
    chained = {}
    cg_in = torch.randn(BATCH, cfg.hidden, device=m.device).to(torch.bfloat16)
    for name, key, kw in (("gate_up", "w_gu", {"epilogue": EPI_SILU_MUL}), ("qkv", "w_qkv", {})):
        wl = [m.w[f"layers.{l}.{key}"] for l in range(cfg.layers)]
        n_out = wl[0].n // 2 if name == "gate_up" else wl[0].n
        outb = torch.empty(BATCH, n_out, dtype=torch.bfloat16, device=m.device)
        side = (torch.empty(BATCH, wl[0].n_extra, dtype=torch.float32, device=m.device)
                if name == "qkv" and wl[0].n_extra else None)
        cs = torch.cuda.Stream(device=m.device)
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for wt in wl:
                ops.gemm(cg_in, wt, outb, side=side, **kw)
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=cs):
                for wt in wl:
                    ops.gemm(cg_in, wt, outb, side=side, **kw)
        torch.cuda.current_stream().wait_stream(cs)
        for _ in range(3):
            cg.replay()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        R = 10
        c0.record()
        for _ in range(R):
            cg.replay()
        c1.record()
        torch.cuda.synchronize()
        us = c0.elapsed_time(c1) * 1000.0 / (R * len(wl))
        nb = (wl[0].n + (wl[0].n_extra if side is not None else 0)) * wl[0].k * 2 + \
            BATCH * wl[0].k * 2 + BATCH * (n_out + (side.shape[1] * 2 if side is not None else 0)) * 2
        chained[name] = {"us_per_launch": round(us, 2), "bytes_per_launch": nb,
                         "GB/s": round(nb / us / 1e3, 1), "frac": round(nb / us / 1e3 / hbm_peak, 4)}
        del cg
    # ---- per-kernel-class device time of an eager step (events around each op)
    with ops.KernelTimer() as kt:
        torch.cuda._sleep(400_000_000)
        dg._step()
    torch.cuda.synchronize()
    dur = kt.durations()
    step_ms_instr = sum(v[0] for v in dur.values())
    kernels = {}
    for cat, (ms, n, _) in sorted(dur.items(), key=lambda kv: -kv[1][0]):
        e = {"ms_per_step": round(ms, 4), "launches": n, "share": round(ms / step_ms_instr, 4)}
        if cat in abytes:
            gbs = abytes[cat] / (ms / 1000.0) / 1e9
            e.update({"GB/s": round(gbs, 1), "frac_hbm": round(gbs / hbm_peak, 4),
                      "bytes_per_step": abytes[cat]})
        kernels[cat] = e
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("gemm_sk_kernel_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(gemm_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(gemm_gbs / hbm_peak, 4), "traffic": traffic,
                "kernel": "gemm_sk_kernel (tcgen05 stream-K decode GEMM, TMA, TMEM)",
                "bytes_per_launch": abytes["gemm"] / (4 * cfg.layers + 1),
                "us_per_launch_in_graph": round(gemm_us / max(gemm_n, 1), 2),
                "peak_source": peak_src,
                "timing": "in-graph exit-to-exit: %globaltimer stamps of every CTA of every launch "
                          "of one replayed decode graph (slx_debug_gemm_trace); a launch costs the "
                          "step from the previous launch's last CTA exit to its own",
                "event_timed_eager_frac": kernels.get("gemm", {}).get("frac_hbm"),
                "chained": dict(chained, method="one CUDA graph of the 32 layers' launches of "
                                "that GEMM back to back (each streams its own layer's weights, "
                                "> L2), CUDA events around 10 replays"),
                "traffic_note": "ncu dram__bytes_read+write per GEMM launch of one step "
                                "(profiles/traffic.json)"}
    lora_ms = max(1e-6, (t_ms - t_nolora_ms) / args.steps)
    lora = {"ms_per_step": round(lora_ms, 4), "backbone_only_ms_per_step": round(t_nolora_ms / args.steps, 4),
            "bytes_moved_per_step": abytes["lora_moved"],
            "GB/s": round(abytes["lora_moved"] / (lora_ms / 1000.0) / 1e9, 1),
            "frac_hbm": round(abytes["lora_moved"] / (lora_ms / 1000.0) / 1e9 / hbm_peak, 4),
            "algorithmic_bytes_per_step": abytes["lora"],
            "method": "in-graph marginal: step time minus the same decode graph on the bare "
                      "backbone (same weights, no LoRA targets); bytes actually moved = every "
                      "slot's stacked A rows streamed by the q/k/v and o GEMMs + the distinct "
                      "adapters' B rows read by the fused expands + the fp32 v side output"}
    return {"value": value, "t_ms": t_ms, "e2e_value": e2e_value, "launches": launches,
            "per_rank": per_rank, "clk": clk.summary(), "roofline": roofline,
            "lora_kernels": lora, "kernels": kernels, "in_graph": in_graph,
            "step_span_us": round(span, 1), "hbm_ledger_gb": hbm_ledger, "distinct": distinct,
            "kernels_per_step": dg.kernels_per_step,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": dg.h2d_bytes(),
                    "d2h_bytes_per_step": dg.d2h_bytes()}}


# ------------------------------------------------------------------------------ ours: prefill
def prefill_flops(cfg, T, n_prompts, L):
    d, f, qd, kvd = cfg.hidden, cfg.ffn, cfg.q_dim, cfg.kv_dim
    gemm = 2 * T * cfg.layers * d * (qd + 2 * kvd + qd + 3 * f) + 2 * n_prompts * d * cfg.vocab
    attn = cfg.layers * n_prompts * (L * (L + 1) // 2) * 4 * cfg.head_dim * cfg.heads
    return gemm, attn


def prefill_gemm_bytes(cfg, T):
    """Algorithmic HBM bytes of one layer's four prefill GEMMs (weights + activations in +
    outputs, residual reads), averaged per GEMM launch."""
    d, f, qd, kvd = cfg.hidden, cfg.ffn, cfg.q_dim, cfg.kv_dim
    qkv = (qd + 2 * kvd) * d * 2 + T * d * 2 + T * (qd + 2 * kvd) * 2
    o = d * qd * 2 + T * qd * 2 + 2 * T * d * 2
    gu = 2 * f * d * 2 + T * d * 2 + T * f * 2
    dn = d * f * 2 + T * f * 2 + 2 * T * d * 2
    return (qkv + o + gu + dn) / 4.0


def run_prefill(steps=3, warmup=1, bare=False, e2e=True, rank=0):
    """BASELINE config 3 on this GPU: 13B shape, 128 adapters r{8,16,64}, 8 x 2048 prompts."""
    import torch

    from paper_2505_14468_b200 import ops
    from paper_2505_14468_b200.config import LLAMA2_13B, LoraConfig
    from paper_2505_14468_b200.model import MultiLoraModel

    cfg = LLAMA2_13B
    rng = np.random.default_rng(0)
    ranks = rng.choice([8, 16, 64], size=N_AD3)
    m = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=P3, max_ctx=L3, n_slots=N_AD3,
                       max_rank=64, max_tokens=P3 * L3)
    m.random_backbone(seed=0)
    for a in range(N_AD3):
        m.pool.load_random(a, LoraConfig(int(ranks[a]), 2.0 * ranks[a]), seed=100 + a)
    slots = rng.choice(N_AD3, size=P3, replace=False)
    dev = m.device
    T = P3 * L3
    h_toks = rng.integers(1, cfg.vocab, size=T).astype(np.int32)
    toks = torch.from_numpy(h_toks).to(dev)
    pos = torch.from_numpy(np.tile(np.arange(L3, dtype=np.int32), P3)).to(dev)
    seq = torch.from_numpy(np.repeat(np.arange(P3, dtype=np.int32), L3)).to(dev)
    slot = torch.from_numpy(np.repeat(slots.astype(np.int32), L3)).to(dev)
    last = torch.from_numpy((np.arange(P3) + 1) * L3 - 1).to(dev)
    segs = [(i * L3, L3, i, 0) for i in range(P3)]
    slot_host = np.repeat(slots.astype(np.int32), L3)
    step = lambda: m.forward(toks, pos, seq, slot, last, segments=segs, slot_host=slot_host)  # noqa: E731
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ops.launch_count()
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"prefill_ms": round(ms, 2), "tokens_per_s": round(T / (ms / 1000.0), 1),
           "gpu_launches": ops.launch_count() - n0}
    # end to end through the public API: host token lists in (H2D), first tokens out (D2H)
    if e2e:
        prompts = [h_toks[i * L3:(i + 1) * L3].tolist() for i in range(P3)]
        ids = slots.tolist()

        def e2e_step():
            seqs, lg = m.prefill(prompts, ids)
            first = m.argmax(lg).cpu()
            for s_ in seqs:
                m.free_seq(s_)
            return first
        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            e2e_step()
        e2e_ms = (time.perf_counter() - t0) * 1000.0 / steps
        out["e2e"] = {"value": round(T / (e2e_ms / 1000.0), 1), "unit": UNIT,
                      "h2d_bytes_per_step": T * 4 * 4 + P3 * 8, "d2h_bytes_per_step": P3 * 4,
                      "ms_per_step": round(e2e_ms, 2),
                      "path": "MultiLoraModel.prefill(host prompts) + argmax + D2H"}
    with ops.KernelTimer() as kt:
        torch.cuda._sleep(200_000_000)
        step()
    torch.cuda.synchronize()
    dur = {k: (round(v[0], 3), v[1]) for k, v in kt.durations().items()}
    _, tf_peak, peak_src = peaks()
    hbm_peak = peaks()[0]
    gemm_flops, attn_flops = prefill_flops(cfg, T, P3, L3)
    g_ms = kt.durations()["gemm"][0]
    a_ms = kt.durations()["attention"][0]
    out["gemm"] = {"ms": round(g_ms, 2), "TFLOP/s": round(gemm_flops / (g_ms / 1000.0) / 1e12, 1),
                   "frac": round(gemm_flops / (g_ms / 1000.0) / 1e12 / tf_peak, 4),
                   "flops": gemm_flops}
    out["attention"] = {"ms": round(a_ms, 2),
                        "TFLOP/s": round(attn_flops / (a_ms / 1000.0) / 1e12, 1),
                        "frac": round(attn_flops / (a_ms / 1000.0) / 1e12 / tf_peak, 4),
                        "flops": attn_flops, "kernel": "flash_prefill (causal)"}
    out["peak_tflops"] = tf_peak
    out["peak_source"] = peak_src
    out["gemm_algorithmic_bytes"] = prefill_gemm_bytes(cfg, T)
    tp = os.path.join(ROOT, "profiles", "prefill_traffic.json")
    if os.path.exists(tp):
        try:
            out["gemm_traffic"] = json.load(open(tp)).get("gemm_tc_dram_bytes_per_launch")
        except (OSError, ValueError):
            pass
    out["kernels_ms"] = dur
    out["adapter_ranks_of_batch"] = [int(ranks[s]) for s in slots]
    # LoRA bytes actually moved (shrink: A of each prompt's adapter for q,k,v,o + x re-read;
    # expand folded into the backbone GEMMs: B as one extra K block per tile)
    l_ms = kt.durations().get("lora", (0.0,))[0]
    out["lora_shrink"] = {"ms": round(l_ms, 2)}
    if bare:
        del m
        torch.cuda.empty_cache()
        m0 = MultiLoraModel(cfg, dtype=torch.bfloat16, max_seqs=P3, max_ctx=L3, n_slots=N_AD3,
                            max_rank=64, max_tokens=P3 * L3, lora_targets=())
        m0.random_backbone(seed=0)
        step0 = lambda: m0.forward(toks, pos, seq, slot, last, segments=segs, slot_host=slot_host)  # noqa: E731
        for _ in range(warmup):
            step0()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            step0()
        e1.record()
        torch.cuda.synchronize()
        ms0 = e0.elapsed_time(e1) / steps
        out["lora_marginal_ms"] = round(ms - ms0, 2)
        out["backbone_only_prefill_ms"] = round(ms0, 2)
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2505_14468_b200._lib import load

    rank, local_rank, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    load()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if rank == 0:
            print(f"[bench] NCCL process group: world={world} backend={dist.get_backend()} "
                  f"ranks=0..{world - 1} (one process per GPU)", file=sys.stderr, flush=True)
    hbm_peak, tf_peak, _ = peaks()
    if args.workload == "config3":
        t0 = time.perf_counter()
        with ClockSampler(local_rank) as clk:
            r = run_prefill(args.steps, args.warmup, bare=not args.no_bare, rank=rank)
        value_local = r["tokens_per_s"]
        if world > 1:
            t = torch.tensor([r["prefill_ms"]], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        else:
            ms = r["prefill_ms"]
        value = world * P3 * L3 / (ms / 1000.0)
        cpu = (cpu_baseline_line("config3", args.ctx)
               if world == 1 and not args.no_cpu_baseline and rank == 0 else None)
        if rank == 0:
            line = {"metric": metric_name("config3", args.ctx), "value": value, "unit": UNIT,
                    "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                    "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                    "dtype": "bf16", "data": "synthetic (random-init 13B-shape weights and adapters)",
                    "config": config_dict("config3", args.ctx, world),
                    "tokens_per_s_per_gpu": value_local,
                    "e2e": r.get("e2e"), "gpu_launches": r.get("gpu_launches"),
                    "roofline": {"bound": "tensor", "achieved": r["gemm"]["TFLOP/s"], "peak": tf_peak,
                                 "unit": "TFLOP/s", "frac": r["gemm"]["frac"],
                                 "traffic": r.get("gemm_traffic"),
                                 "algorithmic_bytes_per_launch": r.get("gemm_algorithmic_bytes"),
                                 "kernel": "gemm_tcp_kernel (persistent tcgen05 prefill GEMM, "
                                           "LoRA fold)",
                                 "traffic_note": "ncu dram__bytes_read+write per prefill GEMM "
                                                 "launch (profiles/prefill_traffic.json)",
                                 "attention": r["attention"]},
                    "prefill": r, "clocks": clk.summary(), "cpu_baseline": cpu,
                    "wall_s": round(time.perf_counter() - t0, 1)}
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    r = run_decode(args, rank, local_rank, world, dist)
    prefill = None
    if not args.no_prefill and world == 1:
        import torch
        torch.cuda.empty_cache()
        prefill = run_prefill(steps=2, warmup=1, bare=False, e2e=False)
    cpu = (cpu_baseline_line("config2", args.ctx)
           if world == 1 and not args.no_cpu_baseline and rank == 0 else None)
    if rank == 0:
        cfgd = config_dict("config2", args.ctx, world)
        line = {
            "metric": metric_name("config2", args.ctx), "value": r["value"], "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["t_ms"] / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init 7B-shape weights and adapters, random tokens)",
            "config": cfgd,
            "run": {"cuda_graph": True, "kernels_per_step": r["kernels_per_step"],
                    "distinct_adapters_in_batch": r["distinct"],
                    "request_routing": "dp.route join-shortest-queue over a global stream of "
                                       f"{BATCH * world} requests"},
            "tokens_per_s_per_gpu": r["value"] / world,
            "per_rank_tokens_per_s": r["per_rank"],
            "e2e": r["e2e"],
            "gpu_launches": r["launches"],
            "roofline": r["roofline"],
            "lora_kernels": r["lora_kernels"],
            "in_graph_us_per_step": r["in_graph"], "step_span_us": r["step_span_us"],
            "kernels": r["kernels"],
            "hbm_ledger_gb": r["hbm_ledger_gb"],
            "prefill_config3": prefill,
            "clocks": r["clk"],
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch(args) -> int:
    """--gpus N outside torchrun: one process per GPU under torch.distributed.run."""
    import socket

    import torch
    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus:
        print(f"bench: --gpus {args.gpus} requested but only {n_vis} GPU(s) visible",
              file=sys.stderr, flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["config2", "config3"], default="config2")
    ap.add_argument("--ctx", type=int, default=128, help="config2: resident context per sequence")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU oracle leg")
    ap.add_argument("--no-prefill", action="store_true", help="config2: skip the config-3 summary")
    ap.add_argument("--no-bare", action="store_true", help="config3: skip the bare-backbone run")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    run_ours(args)


if __name__ == "__main__":
    main()
