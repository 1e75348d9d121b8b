"""Module-layout mirror of ``moeperf.router`` (router.py:22-133): the router
functions of this package, so code written against ``moeperf.router`` only
changes its import.  Arithmetic on the GPU (``stages.py``, ``layer.py``)."""

from .layer import route
from .stages import gate_scores, stable_softmax_row, topk_select
from .types import RoutingResult

__all__ = ["RoutingResult", "gate_scores", "route", "stable_softmax_row", "topk_select"]
