"""CPU: data-parallel routing and pre-loader host logic, incl. world_size-2 gloo runs."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_14468_b200 import dp
from paper_2505_14468_b200.preload import broadcast_groups
from paper_2505_14468_b200.spec import ArtifactKind, Placement, PreloadPlan, TierKind


def _reqs(n=37):
    return [(i, list(range(1 + (i * 7) % 23)), 8 + i % 5) for i in range(n)]


def test_route_balances_and_is_deterministic():
    reqs = _reqs()
    a = dp.route(reqs, 4)
    assert a == dp.route(reqs, 4)
    loads = [0] * 4
    for r, k in zip(reqs, a):
        loads[k] += len(r[1]) + r[2]
    assert max(loads) - min(loads) <= max(len(r[1]) + r[2] for r in reqs)
    shards = [dp.shard(reqs, k, 4) for k in range(4)]
    assert sorted(x[0] for s in shards for x in s) == [r[0] for r in reqs]


def test_broadcast_groups_single_host_read():
    plan = PreloadPlan([
        Placement("llama7b", ArtifactKind.BACKBONE_MODEL, TierKind.GPU, "gpu1"),
        Placement("llama7b", ArtifactKind.BACKBONE_MODEL, TierKind.GPU, "gpu3"),
        Placement("7b-chat", ArtifactKind.ADAPTER_MODEL, TierKind.GPU, "gpu2"),
        Placement("7b-chat", ArtifactKind.ADAPTER_MODEL, TierKind.CONTAINER, "c0"),
        Placement("7b-chat", ArtifactKind.ADAPTER_MODEL, TierKind.GPU, "gpu0"),
    ])
    groups = broadcast_groups(plan, ["gpu0", "gpu1", "gpu2", "gpu3"],
                              lambda p: f"{p.function_id}:{p.kind.value}")
    assert groups == [("7b-chat:adapter_model", 0, [0, 2]), ("llama7b:backbone_model", 1, [1, 3])]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        reqs = _reqs()
        mine = dp.shard(reqs, rank, world)
        # the unique-id exchange the pre-loader's NCCL communicator uses
        obj = [b"uid-from-rank0"] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        allm = dp.gather_metrics({"rank": rank, "n": len(mine), "ids": [r[0] for r in mine]}, world)
        q.put((rank, obj[0], allm))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharding_and_id_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, uid, allm in res:
        assert uid == b"uid-from-rank0"
        ids = sorted(i for m in allm for i in m["ids"])
        assert ids == [r[0] for r in _reqs()]          # every request served exactly once
        assert [m["rank"] for m in allm] == [0, 1]
