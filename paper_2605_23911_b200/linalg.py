"""Module-layout mirror of ``moeperf.linalg`` (linalg.py:22-86).  The
arithmetic (the canonical fp64-fold matmul, the numpy-exact sigmoid / silu)
runs on the GPU (``stages.py``); ``as_matrix`` / ``require_finite`` are the
reference's host-side input coercion and validation."""

from __future__ import annotations

import numpy as np

from .errors import NonFiniteInput, ShapeMismatch
from .stages import dense_matmul, sigmoid, silu

#: Element dtype for all activations and weights (linalg.py:22-23).
DTYPE = np.float32


def as_matrix(a, name: str = "matrix") -> np.ndarray:
    """``linalg.py:27-35``: C-contiguous 2-D float32, else ShapeMismatch."""
    arr = np.asarray(a, dtype=DTYPE)
    if arr.ndim != 2:
        raise ShapeMismatch(f"{name} must be 2-D, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def require_finite(arr, name: str = "input"):
    """``linalg.py:38-42``."""
    if arr.size and not np.isfinite(arr).all():
        raise NonFiniteInput(f"{name} contains non-finite values")
    return arr


def dot_accumulate(a, b):
    """``linalg.py:45-57`` (on the device: one exact fp64 fold per output)."""
    return dense_matmul(a, b)


__all__ = ["DTYPE", "as_matrix", "dense_matmul", "dot_accumulate", "require_finite", "sigmoid", "silu"]
