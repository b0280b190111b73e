"""Artifact pre-loader (§8 row a6): pinned host pool -> HBM, one host read fanned out by NCCL.

The reference materialises a ``PreloadPlan`` GPU placement as ``usable_at_ms = now +
load_from_container_ms | load_cold_ms`` (``/root/reference/pkg/src/slorasim/engine.py:
1040-1053``) with cold-start latency the sequential sum of its parts (``engine.py:189-235``).
Here a placement is a real transfer:

* ``HostArtifactStore`` keeps every artifact (backbone, adapter blobs) in ONE pinned host
  buffer registered once at startup (``cudaHostRegister`` through the C ABI), so a load is a
  DMA with no staging copy;
* ``Preloader.load`` copies an artifact host->device in chunks on a side stream
  (``slx_preload_h2d``) and records an event, so serving overlaps the load;
* ``Preloader.load_broadcast`` reads the host bytes ONCE on the root rank and broadcasts them
  over NVLink to every rank whose GPU holds the placement (``slx_preload_bcast``: chunk i of
  the H2D overlaps the NCCL broadcast of chunk i-1), on a communicator owned by the
  pre-loader alone — the only collective in the system.

``broadcast_groups`` (pure host logic) turns a plan into (artifact, root, receivers) groups.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check
from .spec import TierKind, kind_value

DEFAULT_CHUNK = 64 << 20


@dataclass(frozen=True)
class HostArtifact:
    name: str
    offset: int
    nbytes: int


class HostArtifactStore:
    """All artifacts in one pinned (cudaHostRegister'ed) host buffer, 4 KiB aligned."""

    def __init__(self, capacity_bytes: int, register: bool = True):
        self.capacity = int(capacity_bytes)
        self.buf = np.zeros(self.capacity + 4096, dtype=np.uint8)
        base = self.buf.ctypes.data
        self.base_off = (-base) % 4096
        self.items: dict = {}
        self.used = 0
        self.registered = False
        if register:
            check(_lib.load().slx_host_register(ctypes.c_void_p(base + self.base_off),
                                                self.capacity), "slx_host_register")
            self.registered = True

    def ptr(self, name: str) -> int:
        return self.buf.ctypes.data + self.base_off + self.items[name].offset

    def put(self, name: str, data) -> HostArtifact:
        """Copy a tensor/array's bytes into the store (once, at startup)."""
        if isinstance(data, torch.Tensor):
            raw = data.detach().contiguous().cpu().view(torch.uint8).numpy().reshape(-1)
        else:
            raw = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
        art = self.reserve(name, int(raw.size))
        start = self.base_off + art.offset
        self.buf[start:start + raw.size] = raw
        return art

    def reserve(self, name: str, nbytes: int) -> HostArtifact:
        """Space for an artifact (filled by ``put`` or by a device->host demotion)."""
        off = (self.used + 4095) // 4096 * 4096
        if off + nbytes > self.capacity:
            raise MemoryError(f"host artifact store full ({self.capacity} bytes)")
        art = HostArtifact(name, off, int(nbytes))
        self.items[name] = art
        self.used = off + nbytes
        return art

    def view(self, name: str) -> np.ndarray:
        """The artifact's bytes (host view)."""
        art = self.items[name]
        start = self.base_off + art.offset
        return self.buf[start:start + art.nbytes]

    def close(self) -> None:
        if self.registered:
            check(_lib.load().slx_host_unregister(ctypes.c_void_p(self.buf.ctypes.data + self.base_off)),
                  "slx_host_unregister")
            self.registered = False


def broadcast_groups(plan, gpu_of_rank: list, artifact_name) -> list:
    """Group the GPU placements of a PreloadPlan into broadcasts.

    ``gpu_of_rank[r]`` is the GPU id rank r drives; ``artifact_name(placement)`` names the
    artifact a placement needs.  Returns sorted [(artifact, root_rank, receiver_ranks)] with
    the lowest receiving rank as root, so every artifact is read from host exactly once.
    """
    rank_of = {g: r for r, g in enumerate(gpu_of_rank)}
    need: dict = {}
    for p in plan:
        if kind_value(p.tier) != TierKind.GPU.value or p.instance not in rank_of:
            continue
        need.setdefault(artifact_name(p), set()).add(rank_of[p.instance])
    return sorted((name, min(ranks), sorted(ranks)) for name, ranks in need.items())


class NcclComm:
    """The pre-loader's own NCCL communicator; the unique id is exchanged over the default
    torch.distributed group."""

    def __init__(self, rank: int, world: int):
        lib = _lib.load()
        import torch.distributed as dist
        uid = (ctypes.c_uint8 * lib.slx_nccl_unique_id_bytes())()
        if rank == 0:
            check(lib.slx_nccl_get_unique_id(uid), "slx_nccl_get_unique_id")
        obj = [bytes(uid)] if rank == 0 else [None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], len(obj[0]))
        self.handle = ctypes.c_void_p()
        check(lib.slx_nccl_comm_init(ctypes.byref(self.handle), world, uid, rank), "slx_nccl_comm_init")
        self.rank, self.world = rank, world

    def close(self) -> None:
        if self.handle:
            check(_lib.load().slx_nccl_comm_destroy(self.handle), "slx_nccl_comm_destroy")
            self.handle = ctypes.c_void_p()


class Preloader:
    def __init__(self, store: HostArtifactStore, device, chunk_bytes: int = DEFAULT_CHUNK):
        self.store = store
        self.device = torch.device(device)
        self.chunk = int(chunk_bytes)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.comm_stream = torch.cuda.Stream(device=self.device)

    def load(self, name: str, dst: torch.Tensor | None = None):
        """Async host->device copy of one artifact on the side stream.
        Returns (device uint8 tensor, done event)."""
        art = self.store.items[name]
        if dst is None:
            dst = torch.empty(art.nbytes, dtype=torch.uint8, device=self.device)
        if dst.numel() * dst.element_size() < art.nbytes:
            raise ValueError("destination too small")
        # dst may be a block the caching allocator just recycled from work still queued on the
        # current stream: the copy must not overtake it
        self.copy_stream.wait_stream(torch.cuda.current_stream(self.device))
        ev = torch.cuda.Event(enable_timing=True)
        check(_lib.load().slx_preload_h2d(ctypes.c_void_p(dst.data_ptr()),
                                          ctypes.c_void_p(self.store.ptr(name)), art.nbytes,
                                          self.chunk, ctypes.c_void_p(self.copy_stream.cuda_stream),
                                          None),
              "slx_preload_h2d")
        ev.record(self.copy_stream)
        dst.record_stream(self.copy_stream)
        return dst, ev

    def timed_load_ms(self, name: str, reps: int = 3) -> float:
        """Measured host->HBM load time of an artifact (median), for ArtifactSpec calibration."""
        times = []
        for _ in range(reps):
            start = torch.cuda.Event(enable_timing=True)
            start.record(self.copy_stream)
            _, ev = self.load(name)
            ev.synchronize()
            times.append(start.elapsed_time(ev))
        return float(np.median(times))

    def load_broadcast(self, name: str, root: int, comm: NcclComm,
                       dst: torch.Tensor | None = None, nbytes: int | None = None) -> torch.Tensor:
        """Single host read on ``root``, NVLink fan-out to all ranks of ``comm``.  A receiving
        rank needs the artifact's size: its own store entry, ``nbytes`` or ``dst``."""
        if nbytes is None and name in self.store.items:
            nbytes = self.store.items[name].nbytes
        if dst is None:
            if nbytes is None:
                raise ValueError(f"load_broadcast({name!r}): size unknown on rank {comm.rank} "
                                 "(pass nbytes or dst)")
            dst = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        if comm.rank == root and name not in self.store.items:
            raise KeyError(f"root rank {root} holds no host copy of {name!r}")
        cur = torch.cuda.current_stream(self.device)
        self.copy_stream.wait_stream(cur)
        self.comm_stream.wait_stream(cur)
        src = self.store.ptr(name) if comm.rank == root else None
        check(_lib.load().slx_preload_bcast(ctypes.c_void_p(dst.data_ptr()),
                                            ctypes.c_void_p(src) if src else None,
                                            nbytes if nbytes is not None else dst.numel() * dst.element_size(),
                                            self.chunk, root,
                                            comm.handle,
                                            ctypes.c_void_p(self.copy_stream.cuda_stream),
                                            ctypes.c_void_p(self.comm_stream.cuda_stream)),
              "slx_preload_bcast")
        dst.record_stream(self.comm_stream)
        dst.record_stream(self.copy_stream)
        return dst

    def wait(self) -> None:
        torch.cuda.current_stream(self.device).wait_stream(self.copy_stream)
        torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)


def measure_h2d_gbs(preloader: Preloader, name: str) -> float:
    ms = preloader.timed_load_ms(name)
    return preloader.store.items[name].nbytes / (ms / 1000.0) / 1e9
