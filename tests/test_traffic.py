"""Activation-traffic reports (perfmodel.py:70-180): the package-level
``activation_traffic_closed_form`` / ``traffic_from_traces`` agree with the
reference's own functions (moeperf installed unmodified in baseline/_ref) on
the BASELINE configs, and the two sources agree with each other."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

import paper_2605_23911_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CONFIGS = [  # (E, k, d, f, B)
    (8, 2, 4096, 14336, 512),   # Mixtral-8x7B
    (60, 4, 2048, 1408, 512),   # Qwen2-MoE-60
    (256, 8, 7168, 2048, 512),  # DeepSeek-V3
    (8, 2, 512, 1024, 128),     # small
]


def _moeperf():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "moeperf")):
        pytest.skip("reference not installed in baseline/_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import moeperf

    return moeperf


def _fields(r):
    return (r.unfused_bytes, r.fused_bytes, r.savings_bytes, r.savings_ratio)


def test_closed_form_mixtral_512():
    r = P.activation_traffic_closed_form(1024, 14336, 4096)
    assert (r.unfused_bytes, r.fused_bytes, r.savings_bytes) == (134217728, 37748736, 96468992)
    assert r.source == "closed_form"


@pytest.mark.parametrize("cfg", CONFIGS)
def test_tile_trace_equals_closed_form(cfg):
    e, k, d, f, b = cfg
    counts = np.bincount(np.arange(b * k) % e, minlength=e)
    config = P.ModelConfig(e, k, d, f, P.Gating.SOFTMAX)
    fused = P.trace_from_counts(config, b, counts, P.PipelineParams(fused=True))
    unfused = P.trace_from_counts(config, b, counts, P.PipelineParams(fused=False))
    t = P.traffic_from_traces(fused, unfused)
    c = P.activation_traffic_closed_form(b * k, f, d, config.element_bytes)
    assert _fields(t) == _fields(c)
    assert t.source == "tile_trace"
    with pytest.raises(P.ShapeMismatch):
        P.traffic_from_traces(unfused, fused)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_reports_match_reference(cfg):
    m = _moeperf()
    e, k, d, f, b = cfg
    ours = P.activation_traffic_closed_form(b * k, f, d)
    ref = m.activation_traffic_closed_form(b * k, f, d)
    assert _fields(ours) == (ref.unfused_bytes, ref.fused_bytes, ref.savings_bytes, ref.savings_ratio)
    counts = np.bincount(np.arange(b * k) % e, minlength=e)
    rc = m.ModelConfig(num_experts=e, top_k=k, hidden_dim=d, ffn_dim=f)
    rt = m.traffic_from_traces(m.trace_from_counts(rc, b, counts, m.PipelineParams(fused=True)),
                               m.trace_from_counts(rc, b, counts, m.PipelineParams(fused=False)))
    config = P.ModelConfig(e, k, d, f, P.Gating.SOFTMAX)
    ot = P.traffic_from_traces(P.trace_from_counts(config, b, counts, P.PipelineParams(fused=True)),
                               P.trace_from_counts(config, b, counts, P.PipelineParams(fused=False)))
    assert _fields(ot) == (rt.unfused_bytes, rt.fused_bytes, rt.savings_bytes, rt.savings_ratio)
