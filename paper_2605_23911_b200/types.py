"""Drop-in API types, mirroring the reference's public dataclasses.

Same names, fields, validation rules and error classes as
``moeperf/model.py:14-165`` (ModelConfig, Gating, ExpertWeights, presets),
``moeperf/pipeline.py:63-78`` (PipelineParams), ``moeperf/router.py:21-58``
(RoutingResult) and ``moeperf/scheduler.py:23-75`` (ExpertOffsets,
Permutation, BlockSchedule).  Array fields may hold numpy arrays or torch
tensors (host or CUDA); nothing here computes.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import IndexOutOfRange, ShapeMismatch


class Gating(str, Enum):
    """Gate-score normalisation (``model.py:14-18``)."""

    SOFTMAX = "softmax"
    SIGMOID_NORMALIZED = "sigmoid_normalized"


GATING_CODE = {Gating.SOFTMAX: 0, Gating.SIGMOID_NORMALIZED: 1}


@dataclass(frozen=True)
class ModelConfig:
    """Static shape and routing parameters of one MoE layer (``model.py:21-48``)."""

    num_experts: int
    top_k: int
    hidden_dim: int
    ffn_dim: int
    gating: Gating = Gating.SOFTMAX
    element_bytes: int = 2

    def __post_init__(self) -> None:
        if self.num_experts < 1:
            raise ValueError("num_experts must be >= 1")
        if not 1 <= self.top_k <= self.num_experts:
            raise ValueError(
                f"top_k must be in [1, num_experts], got k={self.top_k} with E={self.num_experts}"
            )
        if self.hidden_dim < 1 or self.ffn_dim < 1:
            raise ValueError("hidden_dim and ffn_dim must be >= 1")
        if self.element_bytes < 1:
            raise ValueError("element_bytes must be >= 1")


#: Published layer shapes (``model.py:52-57``), plus the BASELINE Qwen routed layer.
MODEL_PRESETS: dict[str, ModelConfig] = {
    "Mixtral8x7B": ModelConfig(8, 2, 4096, 14336, Gating.SOFTMAX),
    "Mixtral8x22B": ModelConfig(8, 2, 6144, 16384, Gating.SOFTMAX),
    "DeepSeekV3": ModelConfig(256, 8, 7168, 2048, Gating.SIGMOID_NORMALIZED),
    "Qwen2MoE57B": ModelConfig(64, 4, 3584, 2560, Gating.SOFTMAX),
}


def preset(name: str) -> ModelConfig:
    """Look up a preset by name; ``KeyError`` if unknown (``model.py:60-66``)."""
    try:
        return MODEL_PRESETS[name]
    except KeyError:
        known = ", ".join(sorted(MODEL_PRESETS))
        raise KeyError(f"unknown model preset {name!r}; known: {known}") from None


@dataclass(frozen=True)
class ExpertWeights:
    """Stacked per-expert FFN weights (``model.py:119-165``).

    gate, up: (E*d, f); down: (E*f, d).  Expert e owns rows e*d:(e+1)*d of
    gate/up and e*f:(e+1)*f of down.
    """

    gate: object
    up: object
    down: object

    def validate(self, config: ModelConfig) -> None:
        e, d, f = config.num_experts, config.hidden_dim, config.ffn_dim
        expected = {"gate": (e * d, f), "up": (e * d, f), "down": (e * f, d)}
        for name, want in expected.items():
            got = tuple(getattr(self, name).shape)
            if got != want:
                raise ShapeMismatch(f"{name} weights have shape {got}, expected {want}")

    @classmethod
    def random(cls, config: ModelConfig, rng: np.random.Generator) -> "ExpertWeights":
        """Scaled-normal weights (std 1/sqrt(fan_in)), float32 (``model.py:147-156``)."""
        e, d, f = config.num_experts, config.hidden_dim, config.ffn_dim
        gate = rng.standard_normal((e * d, f)) / np.sqrt(d)
        up = rng.standard_normal((e * d, f)) / np.sqrt(d)
        down = rng.standard_normal((e * f, d)) / np.sqrt(f)
        return cls(gate=gate.astype(np.float32), up=up.astype(np.float32), down=down.astype(np.float32))

    def slice_expert(self, e: int, config: ModelConfig):
        d, f = config.hidden_dim, config.ffn_dim
        return (self.gate[e * d:(e + 1) * d], self.up[e * d:(e + 1) * d], self.down[e * f:(e + 1) * f])


@dataclass(frozen=True)
class PipelineParams:
    """Tile sizes and fusion switch (``pipeline.py:63-78``).

    The sm_100a kernels pick their own tiles; ``block_m`` is used for the
    returned trace (reference accounting), and ``fused`` selects the fused
    gate+up kernel (the only variant on the device path).
    """

    block_m: int = 64
    block_n: int = 64
    block_k: int = 64
    fused: bool = True

    def __post_init__(self) -> None:
        for name in ("block_m", "block_n", "block_k"):
            value = getattr(self, name)
            if not isinstance(value, (int, np.integer)) or isinstance(value, bool):
                raise ValueError(f"{name} must be an integer, got {value!r}")
            if value < 1:
                raise ValueError(f"{name} must be >= 1, got {value}")


@dataclass(frozen=True)
class RoutingResult:
    """Top-k routing decision (``router.py:21-58``): indices (B,k), weights (B,k)."""

    indices: object
    weights: object

    def __post_init__(self) -> None:
        if tuple(self.indices.shape) != tuple(self.weights.shape):
            raise ShapeMismatch(
                f"indices {tuple(self.indices.shape)} and weights {tuple(self.weights.shape)} disagree"
            )
        if len(self.indices.shape) != 2:
            raise ShapeMismatch("routing arrays must be 2-D (B, k)")

    @property
    def num_tokens(self) -> int:
        return int(self.indices.shape[0])

    @property
    def top_k(self) -> int:
        return int(self.indices.shape[1])

    def validate(self, num_experts: int) -> None:
        idx = self.indices
        if int(np.prod(idx.shape)) and (int(idx.min()) < 0 or int(idx.max()) >= num_experts):
            raise IndexOutOfRange(
                f"expert ids must lie in [0, {num_experts}), got range [{int(idx.min())}, {int(idx.max())}]"
            )


@dataclass(frozen=True)
class ExpertOffsets:
    """Exclusive prefix sums of the histogram, length E+1 (``scheduler.py:23-48``)."""

    offsets: object

    def __post_init__(self) -> None:
        if len(self.offsets.shape) != 1 or self.offsets.shape[0] < 1:
            raise ShapeMismatch("offsets must be a 1-D array of length E + 1")

    @property
    def num_experts(self) -> int:
        return int(self.offsets.shape[0]) - 1

    @property
    def total(self) -> int:
        return int(self.offsets[-1])

    def count(self, e: int) -> int:
        return int(self.offsets[e + 1] - self.offsets[e])


@dataclass(frozen=True)
class Permutation:
    """Forward/inverse maps between expanded and expert-major order (``scheduler.py:51-64``)."""

    forward: object
    inverse: object

    def __post_init__(self) -> None:
        if tuple(self.forward.shape) != tuple(self.inverse.shape) or len(self.forward.shape) != 1:
            raise ShapeMismatch("forward/inverse must be 1-D and equal length")


@dataclass(frozen=True)
class BlockSchedule:
    """Flat list of ``(expert_id, expert-local row offset)`` tiles (``scheduler.py:67-75``)."""

    entries: tuple
    block_m: int

    def __len__(self) -> int:
        return len(self.entries)
