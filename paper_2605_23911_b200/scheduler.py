"""Module-layout mirror of ``moeperf.scheduler`` (scheduler.py:24-117).
Histogram and permutation run on the GPU (``stages.py``); offsets and the
block schedule are E-sized host metadata, as in the reference."""

from .stages import build_permutation, expert_histogram
from .trace import build_block_schedule, expert_offsets
from .types import BlockSchedule, ExpertOffsets, Permutation

__all__ = ["BlockSchedule", "ExpertOffsets", "Permutation", "build_block_schedule", "build_permutation",
           "expert_histogram", "expert_offsets"]
