"""Reactive GPU offloading with real memory moves (§8 f2).

The reference decides which GPU-resident artifacts leave when an incoming batch does not
fit (``/root/reference/pkg/src/slorasim/offload.py:89-194``) and books the move in its
ledger (``offload.py:198-226``): GPU bytes are released at once and a demoted model
becomes usable in its container after ``size / demotion_gbps`` (``engine.py:76``).

* ``select_evictions`` is the same policy, decision for decision (differential test against
  the reference in ``tests/test_offload.py``): candidates in ascending value density (ties:
  smaller value, larger weight, function id, kind); functions being invoked are protected;
  a model leaves only together with its dependents on that GPU (its kernel; for a backbone,
  every adapter of the family and their kernels), whose bytes count toward the freed total;
  a function's context overhead is freed with its last process-holding artifact; models are
  demoted to the attached container with the most room that fits, everything else is
  discarded.
* ``Offloader.apply`` turns the decisions into memory moves on this GPU: an adapter slot's
  blob is copied device -> pinned host (``slx_offload_d2h``, chunked, side stream) into the
  container tier (a ``HostArtifactStore``) and its slot evicted (HBM returned to the
  allocator once the copy has drained); a backbone demotion copies every packed weight.
  The measured copy time replaces ``size / demotion_gbps``.  ``Offloader.promote`` brings a
  demoted adapter back through the pre-loader (pinned host -> HBM).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

import torch

from . import _lib
from ._lib import check
from .spec import ArtifactKind, kind_value

_MODELS = (ArtifactKind.BACKBONE_MODEL.value, ArtifactKind.ADAPTER_MODEL.value)
_KERNEL = ArtifactKind.KERNEL.value
_ADAPTER = ArtifactKind.ADAPTER_MODEL.value
_BACKBONE = ArtifactKind.BACKBONE_MODEL.value


class InsufficientEvictableMemory(Exception):
    """Not enough unprotected resident bytes (reference ``offload.py:19``)."""


class StaleStateError(Exception):
    """The residency changed between selection and application (``offload.py:23``)."""


@dataclass(frozen=True)
class OffloadRequest:
    gpu_id: str
    required_bytes: int
    protected: frozenset = frozenset()

    def __post_init__(self):
        object.__setattr__(self, "protected", frozenset(self.protected))
        if self.required_bytes <= 0:
            raise ValueError("required_bytes must be > 0")


@dataclass(frozen=True)
class ResidentValue:
    function_id: str
    kind: object
    weight: int
    value: float

    @property
    def density(self) -> float:
        return self.value / self.weight


class Eviction(NamedTuple):
    function_id: str
    kind: object
    gpu_id: str
    size_bytes: int
    destination: str   # "discard" or a container id


def _adapters_of(catalog, backbone_fid: str):
    if hasattr(catalog, "adapters_of"):
        return catalog.adapters_of(backbone_fid)
    return [f for f in catalog if getattr(f, "backbone_id", None) == backbone_fid]


def select_evictions(request: OffloadRequest, resident: list, catalog, free_bytes: int = 0,
                     container_free: dict | None = None,
                     context_overhead_bytes: int = 0) -> list:
    """Evictions freeing at least ``required_bytes - free_bytes`` on ``request.gpu_id`` with
    minimal value lost (reference ``offload.py:89-194``; same arguments and errors)."""
    need = request.required_bytes - free_bytes
    if need <= 0:
        return []
    order = sorted(resident, key=lambda r: (r.value / r.weight, r.value, -r.weight,
                                            r.function_id, kind_value(r.kind)))
    by_key = {(r.function_id, kind_value(r.kind)): r for r in order}
    # kinds each function still holds on this GPU (context overhead goes with the last
    # artifact that keeps a process alive; a bare backbone needs none)
    held: dict = {}
    for r in order:
        held.setdefault(r.function_id, set()).add(kind_value(r.kind))

    picked: list = []
    taken: set = set()
    freed = 0

    def release(r, kv: str) -> None:
        nonlocal freed
        if (r.function_id, kv) in taken:
            return
        taken.add((r.function_id, kv))
        picked.append((r, kv))
        extra = 0
        if context_overhead_bytes:
            now = held[r.function_id]
            after = now - {kv}
            alive_now = bool(now) and now != {_BACKBONE}
            alive_after = bool(after) and after != {_BACKBONE}
            if alive_now and not alive_after:
                extra = context_overhead_bytes
            now.discard(kv)
        freed += r.weight + extra

    for r in order:
        if freed >= need:
            break
        kv = kind_value(r.kind)
        if (r.function_id, kv) in taken or r.function_id in request.protected:
            continue
        if kv in _MODELS:
            deps = []
            k = by_key.get((r.function_id, _KERNEL))
            if k is not None:
                deps.append((k, _KERNEL))
            if kv == _BACKBONE:
                for ad in _adapters_of(catalog, r.function_id):
                    a = by_key.get((ad.id, _ADAPTER))
                    if a is not None:
                        deps.append((a, _ADAPTER))
                        ak = by_key.get((ad.id, _KERNEL))
                        if ak is not None:
                            deps.append((ak, _KERNEL))
            if any(d.function_id in request.protected for d, _ in deps):
                continue
            for d, dkv in deps:
                release(d, dkv)
        release(r, kv)
    if freed < need:
        raise InsufficientEvictableMemory(f"gpu {request.gpu_id}: can free {freed} of {need} bytes")

    room = dict(container_free or {})
    out = []
    for r, kv in picked:
        dest = "discard"
        if kv in _MODELS and room:
            for cid in sorted(room, key=lambda c: (-room[c], c)):
                if room[cid] >= r.weight:
                    dest = cid
                    room[cid] -= r.weight
                    break
        out.append(Eviction(r.function_id, r.kind, request.gpu_id, r.weight, dest))
    return out


class Offloader:
    """Materialises evictions on ONE GPU's model.

    ``adapter_slot``: function id -> adapter slot of ``model.pool``; ``backbone_fid``: the
    function id of the model's backbone.  ``store`` is the container tier (pinned host)."""

    def __init__(self, model, store, adapter_slot: dict, backbone_fid: str | None = None,
                 chunk_bytes: int = 64 << 20):
        self.model, self.store = model, store
        self.adapter_slot = dict(adapter_slot)
        self.backbone_fid = backbone_fid
        self.chunk = int(chunk_bytes)
        self.stream = torch.cuda.Stream(device=model.device)
        self.demoted: dict = {}   # function id -> (container id, store name, LoraConfig | None)

    def _d2h(self, name: str, src: torch.Tensor) -> torch.cuda.Event:
        nbytes = src.numel() * src.element_size()
        if name not in self.store.items:
            self.store.reserve(name, nbytes)
        if self.store.items[name].nbytes != nbytes:
            raise ValueError(f"{name}: container copy has a different size")
        self.stream.wait_stream(torch.cuda.current_stream(self.model.device))
        check(_lib.load().slx_offload_d2h(ctypes.c_void_p(self.store.ptr(name)),
                                          ctypes.c_void_p(src.data_ptr()), nbytes, self.chunk,
                                          ctypes.c_void_p(self.stream.cuda_stream), None),
              "slx_offload_d2h")
        src.record_stream(self.stream)   # HBM reused only after the copy drained
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        return ev

    def apply(self, evictions: list) -> list:
        """Evict / demote; returns [(measured demotion ms, eviction)] like the reference's
        ``apply_evictions`` (0 for discards).  Raises StaleStateError for artifacts that are
        no longer resident here."""
        pool = self.model.pool
        for ev in evictions:
            kv = kind_value(ev.kind)
            if kv == _ADAPTER and (ev.function_id not in self.adapter_slot
                                   or pool.blobs[self.adapter_slot[ev.function_id]] is None):
                raise StaleStateError(f"{ev.function_id}/adapter not resident")
            if kv == _BACKBONE and (ev.function_id != self.backbone_fid or not self.model.w):
                raise StaleStateError(f"{ev.function_id}/backbone not resident")
        done = []
        for ev in evictions:
            kv = kind_value(ev.kind)
            start = torch.cuda.Event(enable_timing=True)
            start.record(self.stream)
            end = None
            if kv == _ADAPTER:
                slot = self.adapter_slot[ev.function_id]
                blob, cfg = pool.blobs[slot], pool.configs[slot]
                if ev.destination != "discard":
                    end = self._d2h(f"offload/{ev.function_id}", blob)
                    self.demoted[ev.function_id] = (ev.destination, f"offload/{ev.function_id}", cfg)
                pool.evict(slot)
                del blob
            elif kv == _BACKBONE:
                if ev.destination != "discard":
                    for k, t in self.model.w.items():
                        end = self._d2h(f"offload/{ev.function_id}/{k}", getattr(t, "data", t))
                    self.demoted[ev.function_id] = (ev.destination, f"offload/{ev.function_id}", None)
                self.model.w = {}
            done.append((start, end, ev))
        out = []
        for start, end, ev in done:
            if end is None:
                out.append((0.0, ev))
            else:
                end.synchronize()
                out.append((start.elapsed_time(end), ev))
        return out

    def promote(self, function_id: str, preloader) -> torch.cuda.Event:
        """A demoted adapter back into its slot: pinned host -> HBM through the pre-loader."""
        _, name, cfg = self.demoted[function_id]
        if cfg is None:
            raise ValueError("promote: only adapters are re-installed in place")
        dst, ev = preloader.load(name)
        preloader.wait()
        self.model.pool.install(self.adapter_slot[function_id], dst.view(torch.bfloat16), cfg)
        del self.demoted[function_id]
        return ev
