"""Domain types of the hot path, mirroring the reference's public Python interface.

Same names, fields, defaults and validation errors as the reference value objects the
multi-LoRA path consumes (``/root/reference/pkg/src/slorasim/core.py``):

* ``ArtifactKind`` / ``TierKind`` (``core.py:24-53``)
* ``ArtifactSpec`` (``core.py:56-78``): size + cold / container-promotion load times
* ``FunctionSpec`` (``core.py:81-125``): the latency law ``T0 + alpha*(b-1)``, decode
  ms/token and KV bytes per request the B200 runtime calibrates (``calibrate.py``)
* ``Placement`` / ``PreloadPlan`` (``core.py:222-262``): what the pre-loader materialises

Every function in this package also accepts the reference's own objects (duck typing on
the same attribute names), so either can be passed across the boundary.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class ConfigError(Exception):
    """Raised when a spec violates an invariant (reference ``core.py:17``)."""


class ArtifactKind(Enum):
    LIBRARY = "library"
    BACKBONE_MODEL = "backbone_model"
    ADAPTER_MODEL = "adapter_model"
    KERNEL = "kernel"

    @property
    def is_model(self) -> bool:
        return self in (ArtifactKind.BACKBONE_MODEL, ArtifactKind.ADAPTER_MODEL)


class TierKind(Enum):
    CONTAINER = "container"
    GPU = "gpu"


@dataclass(frozen=True)
class ArtifactSpec:
    kind: ArtifactKind
    size_bytes: int
    load_cold_ms: float
    load_from_container_ms: float = 0.0

    def __post_init__(self):
        if self.size_bytes <= 0:
            raise ConfigError(f"artifact size_bytes must be > 0, got {self.size_bytes}")
        if self.load_from_container_ms < 0 or self.load_cold_ms < self.load_from_container_ms:
            raise ConfigError("need load_cold_ms >= load_from_container_ms >= 0, got "
                              f"{self.load_cold_ms} / {self.load_from_container_ms}")


@dataclass(frozen=True)
class FunctionSpec:
    id: str
    artifacts: tuple
    slo_ttft_ms: float
    prefill_base_ms: float
    prefill_marginal_ms: float = 0.0
    decode_ms_per_token: float = 0.0
    kv_cache_bytes_per_request: int = 0
    container_init_ms: float = 0.0
    backbone_id: str | None = None

    def __post_init__(self):
        if isinstance(self.artifacts, list):
            object.__setattr__(self, "artifacts", tuple(self.artifacts))
        if self.prefill_base_ms <= 0:
            raise ConfigError(f"{self.id}: prefill_base_ms must be > 0")
        if self.prefill_marginal_ms < 0:
            raise ConfigError(f"{self.id}: prefill_marginal_ms must be >= 0")
        if self.slo_ttft_ms <= self.prefill_base_ms:
            raise ConfigError(f"{self.id}: slo_ttft_ms must exceed prefill_base_ms")
        kinds = [a.kind for a in self.artifacts]
        n_adapter = sum(1 for k in kinds if k is ArtifactKind.ADAPTER_MODEL)
        n_backbone = sum(1 for k in kinds if k is ArtifactKind.BACKBONE_MODEL)
        if self.backbone_id is not None:
            if n_adapter != 1:
                raise ConfigError(f"{self.id}: adapter function needs exactly one adapter_model artifact")
            if n_backbone != 0:
                raise ConfigError(f"{self.id}: adapter function must not own a backbone_model artifact")
        elif n_backbone > 1:
            raise ConfigError(f"{self.id}: at most one backbone_model artifact")

    @property
    def is_adapter(self) -> bool:
        return self.backbone_id is not None

    def artifact(self, kind: ArtifactKind):
        for a in self.artifacts:
            if a.kind is kind:
                return a
        return None


@dataclass(frozen=True)
class Placement:
    function_id: str
    kind: ArtifactKind
    tier: TierKind
    instance: str

    def __post_init__(self):
        if self.kind is ArtifactKind.LIBRARY and self.tier is not TierKind.CONTAINER:
            raise ConfigError("library placements are container-tier only")
        if self.kind is ArtifactKind.KERNEL and self.tier is not TierKind.GPU:
            raise ConfigError("kernel placements are GPU-tier only")

    def sort_key(self):
        return (self.function_id, self.kind.value, self.tier.value, self.instance)


@dataclass(frozen=True)
class PreloadPlan:
    placements: frozenset = frozenset()

    def __post_init__(self):
        object.__setattr__(self, "placements", frozenset(self.placements))

    def __iter__(self):
        return iter(sorted(self.placements, key=Placement.sort_key))

    def __len__(self):
        return len(self.placements)

    def on_instance(self, tier: TierKind, instance: str) -> list:
        return [p for p in self if p.tier is tier and p.instance == instance]


def kind_value(kind) -> str:
    """Enum value of either this package's or the reference's ArtifactKind/TierKind."""
    return getattr(kind, "value", kind)
