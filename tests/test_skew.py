"""Routing-skew generator (paper_2605_23911_b200/skew.py) against fixtures
drawn by the reference harness itself (tests/golden/make_skew_golden.py)."""

from __future__ import annotations

import ast
import json
import os

import numpy as np
import pytest

from golden_util import bits_equal
from paper_2605_23911_b200 import errors
from paper_2605_23911_b200.skew import (SkewSpec, imbalance_metrics, load_routing, save_routing,
                                        synthesize_routing, zipf_probabilities)
from paper_2605_23911_b200.types import Gating, ModelConfig

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "skew_golden.npz")


@pytest.fixture(scope="module")
def skew_golden():
    z = np.load(GOLD)
    return {k: z[k] for k in z.files}


def test_synthesize_routing_matches_reference_draws(skew_golden):
    cases = [ast.literal_eval(str(m)) for m in skew_golden["meta"]]
    for n, (dist, alpha, seed, B, E, k) in enumerate(cases):
        cfg = ModelConfig(E, k, 64, 64, Gating.SOFTMAX)
        r = synthesize_routing(SkewSpec(dist, alpha, seed, B, cfg))
        bits_equal(r.indices, skew_golden[f"c{n}/indices"])
        bits_equal(r.weights, skew_golden[f"c{n}/weights"])
        counts = np.bincount(r.indices.reshape(-1), minlength=E)
        m = imbalance_metrics(counts)
        np.testing.assert_array_equal([m.max_over_mean, m.gini, m.active_experts], skew_golden[f"c{n}/metrics"])
        if alpha is not None:
            bits_equal(zipf_probabilities(E, alpha), skew_golden[f"c{n}/probs"])
        # every token's experts are distinct
        assert all(len(set(row)) == k for row in r.indices.tolist())


def test_spec_validation_and_alpha_zero():
    cfg = ModelConfig(64, 2, 64, 64, Gating.SOFTMAX)
    with pytest.raises(errors.InvalidSpec):
        SkewSpec("zipf", 0.0, 0, 8, cfg)
    with pytest.raises(errors.InvalidSpec):
        SkewSpec("uniform", 1.0, 0, 8, cfg)
    with pytest.raises(errors.InvalidSpec):
        SkewSpec("pareto", None, 0, 8, cfg)
    assert SkewSpec.for_alpha(0, 3, 8, cfg).distribution == "uniform"
    with pytest.raises(errors.AllZero):
        imbalance_metrics(np.zeros(4, np.int64))


def test_routing_json_roundtrip(tmp_path):
    cfg = ModelConfig(16, 2, 64, 64, Gating.SOFTMAX)
    spec = SkewSpec("zipf", 1.2, 9, 33, cfg)
    r = synthesize_routing(spec)
    p = tmp_path / "routing.json"
    save_routing(p, r, spec)
    r2 = load_routing(p)
    bits_equal(r2.indices, r.indices)
    bits_equal(r2.weights, r.weights)
    assert json.loads(p.read_text())["spec"]["alpha"] == 1.2
    with pytest.raises(errors.ShapeMismatch):
        from paper_2605_23911_b200.skew import routing_from_dict
        routing_from_dict({"indices": [1, 2], "weights": [0.5, 0.5]})
