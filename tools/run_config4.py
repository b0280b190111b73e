"""Config 4 system replay through the UNCHANGED reference simulator.

Two backbone families (Llama-2-7B / -13B shapes) with K adapter functions each, a bursty trace
(reference workload.generate_trace(BURSTY), retry-next-seed when a function id is unreachable,
SURVEY §0.9), contention-aware batching + offload on (reference SimConfig defaults), on an 8 x B200
cluster (180 GB HBM each, two host containers per GPU).  Runs slorasim.run twice:
  * "paper":  the reference's desk-scale FunctionSpecs (profiles.py: 500/100 ms, 10 ms/token, ...)
  * "b200":   the same catalog with T0 / alpha / decode ms / KV bytes / host->HBM loads replaced
              by the values measured on B200 with this repo's kernels (profiles/r01_calibrated_specs.json,
              written by tools/calibrate_b200.py); remote-storage cold fetches (2 GB/s) are kept.
The simulator is imported from /root/reference (CPU only; not used on the GPU box).
SLOs follow the reference rule: 5x the warm prefill (profiles.py:28).
python tools/run_config4.py [--adapters 8] [--duration 120] [--rate 0.05 0.1 0.3] [--replan-period 10]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
from slorasim import metrics, profiles, workload  # noqa: E402
from slorasim.core import FunctionCatalog, parse_cluster, parse_function  # noqa: E402
from slorasim.engine import SimConfig, run  # noqa: E402

PAPER = {  # reference profiles.py DEFAULT_FUNCTIONS_YAML
    "llama7b": dict(pb=500.0, pm=100.0, dec=10.0, kv=100_000_000, bb=14_000_000_000, bb_cold=7000.0,
                    bb_hot=280.0, ad=200_000_000, ad_cold=100.0, ad_hot=4.0),
    "llama13b": dict(pb=800.0, pm=160.0, dec=15.0, kv=150_000_000, bb=26_000_000_000, bb_cold=13000.0,
                     bb_hot=520.0, ad=200_000_000, ad_cold=100.0, ad_hot=4.0),
}


def b200_params(cal):
    out = {}
    for fam, p in PAPER.items():
        c = cal["functions"][fam]
        q = dict(p)
        q.update(pb=c["prefill_base_ms"], pm=c["prefill_marginal_ms"],
                 dec=max(c["decode_ms_per_token_b1"], c["decode_step_ms_b16"]),
                 kv=int(c["kv_bytes_per_request"]), bb=int(c["backbone_bytes"]),
                 bb_cold=c["backbone_bytes"] / 2e9 * 1e3, bb_hot=c["backbone_load_ms"],
                 ad=int(c["adapter_bytes"]), ad_cold=c["adapter_bytes"] / 2e9 * 1e3,
                 ad_hot=c["adapter_load_ms"])
        out[fam] = q
    return out


def catalog(params, k):
    fns = []
    for fam, p in params.items():
        common = dict(slo_ttft_ms=5.0 * p["pb"], prefill_base_ms=p["pb"], prefill_marginal_ms=p["pm"],
                      decode_ms_per_token=p["dec"], kv_bytes_per_request=p["kv"], container_init_ms=800)
        lib = {"kind": "library", "size_bytes": 2_000_000_000, "load_cold_ms": 1000}
        ker = {"kind": "kernel", "size_bytes": 500_000_000, "load_cold_ms": 500}
        fns.append(dict(id=fam, artifacts=[lib, {"kind": "backbone", "size_bytes": p["bb"],
                   "load_cold_ms": p["bb_cold"], "load_from_container_ms": p["bb_hot"]}, ker], **common))
        for i in range(k):
            fns.append(dict(id=f"{fam[5:]}-a{i:02d}", backbone=fam, artifacts=[lib, {
                "kind": "adapter", "size_bytes": p["ad"], "load_cold_ms": p["ad_cold"],
                "load_from_container_ms": p["ad_hot"]}, ker], **common))
    return FunctionCatalog([parse_function(f) for f in fns])


def cluster(n_gpus=8):
    return parse_cluster({
        "context_overhead_bytes": profiles.CONTEXT_OVERHEAD_BYTES,
        "gpus": [{"id": f"gpu{g}", "mem_bytes": 180_000_000_000} for g in range(n_gpus)],
        "containers": [{"id": f"host{g}{s}", "mem_bytes": 240_000_000_000, "gpu": f"gpu{g}"}
                       for g in range(n_gpus) for s in "ab"]})


def bursty_trace(fids, duration_s, rate, seed):
    traces, retries = [], 0
    for fid in sorted(fids):
        for attempt in range(50):
            try:
                traces.append(workload.generate_trace(workload.CovClass.BURSTY, duration_s, rate,
                                                      seed + attempt, function_id=fid))
                break
            except workload.ClassUnreachable:
                retries += 1
        else:
            raise RuntimeError(f"{fid}: bursty class unreachable")
    return workload.merge_traces(traces), retries


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--adapters", type=int, default=8)
    ap.add_argument("--duration", type=float, default=120.0)
    ap.add_argument("--rate", type=float, nargs="+", default=[0.05, 0.1, 0.3])
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--replan-period", type=float, default=10.0,
                    help="SimConfig.replan_period_s (reference default 10 s; SURVEY 8d: raise it at 130 fns)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_config4_sim.json"))
    ap.add_argument("--cal", default=os.path.join(ROOT, "profiles", "r01_calibrated_specs.json"),
                    help="calibrated specs written by tools/calibrate_b200.py")
    a = ap.parse_args()
    cal = json.load(open(a.cal))
    print("calibration:", a.cal, flush=True)
    cl = cluster(a.gpus)
    res = {"setup": {"adapters_per_family": a.adapters, "functions": 2 * (a.adapters + 1),
                     "gpus": a.gpus, "gpu_mem_bytes": 180e9, "duration_s": a.duration,
                     "trace": "BURSTY (reference generate_trace)",
                     "sim": "reference slorasim.run, SimConfig defaults (offload, preload, sharing on)",
                     "replan_period_s": a.replan_period,
                     "calibration_device": cal["device"]}, "runs": {}}
    for rate, name, params in [(r, n, p) for r in a.rate
                               for n, p in (("paper", PAPER), ("b200", b200_params(cal)))]:
        cat = catalog(params, a.adapters)
        trace, retries = bursty_trace([f.id for f in cat], a.duration, rate, a.seed)
        t0 = time.time()
        result = run(SimConfig(seed=a.seed, replan_period_s=a.replan_period), cl, cat, trace)
        rep = metrics.build_report(name, result, profiles.default_pricing())
        o = rep.overall
        res["runs"][f"{name}@{rate}"] = {
            "spec": name, "requested_rate_per_fn": rate, "params": params, "requests": o.requests, "realized_rate_per_fn":
                len(trace.records) / a.duration / len(cat),
            "trace_retries": retries,
            "ttft_mean_ms": o.ttft_mean_ms, "ttft_p50_ms": o.ttft_p50_ms, "ttft_p90_ms": o.ttft_p90_ms,
            "ttft_p99_ms": o.ttft_p99_ms, "tpot_mean_ms": o.tpot_mean_ms, "e2e_mean_ms": o.e2e_mean_ms,
            "slo_violation_rate": o.slo_violation_rate, "tokens_per_s": rep.tokens_per_s,
            "requests_per_s": rep.requests_per_s, "peak_batch_size": rep.peak_batch_size,
            "monetary_cost": rep.monetary_cost, "cold_breakdown_totals": o.cold_breakdown_totals,
            "sim_wall_s": time.time() - t0}
        print(name, rate, json.dumps({k: v for k, v in res["runs"][f"{name}@{rate}"].items() if k != "params"}), flush=True)
    json.dump(res, open(a.out, "w"), indent=1, default=str)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
