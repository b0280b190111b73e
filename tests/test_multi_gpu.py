"""Multi-GPU legs: the pre-loader's single host read + NCCL fan-out at world size 2
(reference: the planner's GPU placements become usable at ``now + load_ms``,
/root/reference/pkg/src/slorasim/engine.py:1036-1053, with one backbone per GPU,
ledger.py:130-134) and ``bench.py --gpus N`` as the driver launches it.  The GPU cases skip on
boxes with fewer than two GPUs; the CPU case checks that an impossible ``--gpus`` fails loudly."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _bcast_worker(rank, world, port, nbytes, q):
    import torch.distributed as dist

    from paper_2505_14468_b200.preload import HostArtifactStore, NcclComm, Preloader
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = NcclComm(rank, world)
        store = HostArtifactStore(nbytes + (1 << 20))
        if rank == 0:   # the single host copy lives on the root only
            store.put("artifact", np.random.default_rng(7).integers(0, 256, nbytes, dtype=np.uint8))
        pre = Preloader(store, torch.device("cuda", rank), chunk_bytes=1 << 20)
        dst = pre.load_broadcast("artifact", 0, comm, nbytes=nbytes)
        pre.wait()
        torch.cuda.synchronize()
        got = dst.cpu().numpy()
        ref = np.random.default_rng(7).integers(0, 256, nbytes, dtype=np.uint8)
        q.put((rank, bool(np.array_equal(got, ref))))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_preload_broadcast_world2_bit_identical():
    """One pinned host read on rank 0, chunked H2D overlapped with ncclBroadcast to rank 1: both
    GPUs hold the artifact bit-for-bit (odd size: a partial last chunk)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    nbytes = (5 << 20) + 12345
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, nbytes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


@pytest.mark.gpu
def test_bench_two_gpus_prints_one_line_with_n_gpus_2():
    """``bench.py --gpus 2`` outside torchrun launches one process per GPU (NCCL) and rank 0
    prints one JSON line with n_gpus = 2 and the whole-job value."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline", "--no-prefill"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    assert len(lines[0]["per_rank_tokens_per_s"]) == 2
    assert "NCCL process group: world=2" in r.stderr


def test_bench_more_gpus_than_visible_fails_loudly():
    """CPU box: asking for more GPUs than are visible is an error, not a silent 1-GPU run."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n + 2), "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "requested but only" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
