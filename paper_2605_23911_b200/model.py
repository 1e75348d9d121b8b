"""Module-layout mirror of ``moeperf.model`` (model.py:14-165): the layer
configuration and weight containers of the drop-in API."""

from .types import MODEL_PRESETS, ExpertWeights, Gating, ModelConfig, preset

__all__ = ["MODEL_PRESETS", "ExpertWeights", "Gating", "ModelConfig", "preset"]
