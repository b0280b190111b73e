"""Data-parallel sharding across the GPUs of one node (§8 row e).

Inference needs no collective: every rank holds a full backbone replica and an adapter pool,
and requests are partitioned across ranks.  The reference's router (``engine.py:501-544``)
pins a backbone family to the GPU already holding it; with a replica on every GPU the router
here balances load instead: deterministic join-shortest-queue on outstanding tokens, so
every rank computes the same assignment from the same request stream with no exchange.
The only collectives are out-of-band: the pre-loader's NCCL broadcast (preload.py) and an
end-of-run gather of metrics (``gather_metrics``).
"""

from __future__ import annotations


def route(requests, world: int, cost=lambda r: len(r[1]) + r[2]) -> list:
    """Assign requests [(request_id, prompt, max_new_tokens, ...)] to ranks.
    Returns the rank of each request (join-shortest-queue on outstanding tokens,
    ties -> lowest rank); identical on every rank."""
    load = [0] * world
    out = []
    for r in requests:
        k = min(range(world), key=lambda i: (load[i], i))
        out.append(k)
        load[k] += cost(r)
    return out


def shard(requests, rank: int, world: int, **kw) -> list:
    assign = route(requests, world, **kw)
    return [r for r, k in zip(requests, assign) if k == rank]


def gather_metrics(local: dict, world: int) -> list:
    """All ranks' metric dicts on every rank (torch.distributed object all-gather)."""
    if world == 1:
        return [local]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, local)
    return out
