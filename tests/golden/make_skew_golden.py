"""Golden routing tables from the REFERENCE skew harness (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_skew_golden.py

Each case is (distribution, alpha, seed, num_tokens, E, k); the fixture
stores the reference's indices, weights and imbalance metrics.
"""

from __future__ import annotations

import os

import numpy as np

from moeperf import Gating, ModelConfig  # reference package, from PYTHONPATH
from moeperf.scheduler import expert_histogram
from moeperf.skew import SkewSpec, imbalance_metrics, synthesize_routing, zipf_probabilities

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [
    ("uniform", None, 0, 512, 64, 2),
    ("zipf", 0.5, 1, 512, 64, 2),
    ("zipf", 0.8, 2, 512, 64, 2),
    ("zipf", 1.2, 3, 512, 64, 2),
    ("zipf", 1.6, 4, 512, 64, 2),
    ("zipf", 2.0, 5, 512, 64, 2),
    ("zipf", 1.0, 6, 40, 8, 3),
    ("zipf", 6.0, 7, 16, 4, 4),   # k == E with extreme skew: rejection + completion path
]

out = {}
for n, (dist, alpha, seed, B, E, k) in enumerate(CASES):
    cfg = ModelConfig(E, k, 64, 64, Gating.SOFTMAX)
    r = synthesize_routing(SkewSpec(dist, alpha, seed, B, cfg))
    m = imbalance_metrics(expert_histogram(r, E))
    out[f"c{n}/indices"] = r.indices
    out[f"c{n}/weights"] = r.weights
    out[f"c{n}/metrics"] = np.array([m.max_over_mean, m.gini, m.active_experts], np.float64)
    if alpha is not None:
        out[f"c{n}/probs"] = zipf_probabilities(E, alpha)
out["meta"] = np.array([repr(c) for c in CASES])
np.savez_compressed(os.path.join(HERE, "skew_golden.npz"), **out)
print("wrote", len(CASES), "cases")
