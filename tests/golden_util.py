"""Helpers shared by the test modules (kept out of conftest so they import by name)."""

from __future__ import annotations

import ast

import numpy as np


def golden_meta(golden):
    return [ast.literal_eval(str(m)) for m in golden["meta"]]


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.dtype.kind == "f":
        assert a.dtype == b.dtype, (a.dtype, b.dtype)
        view = np.uint32 if a.dtype == np.float32 else np.uint64
        np.testing.assert_array_equal(a.view(view), b.view(view))
    else:
        np.testing.assert_array_equal(a, b)
