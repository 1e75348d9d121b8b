"""Generate golden fixtures by running the REFERENCE itself (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are not stored: every case records its generator (seed + shape), and
the tests regenerate the identical inputs with ``oracle.moe_oracle``'s
PCG64 generators (the same draw order as the reference's
``tests/conftest.py:37-58``).  Outputs come from ``moeperf`` (the reference
package), so the fixtures pin both the oracle restatement and the CUDA path.
/root/reference is read-only and absent on the GPU box; only the .npz files
travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import moeperf  # noqa: E402  (reference package, from PYTHONPATH)
from moeperf import ExpertWeights, Gating, ModelConfig, PipelineParams  # noqa: E402
from moeperf.pipeline import dense_moe_oracle, moe_forward  # noqa: E402
from moeperf.router import route, topk_select  # noqa: E402
from moeperf.scheduler import build_permutation, expert_histogram  # noqa: E402

from oracle.moe_oracle import make_instance, make_router_instance  # noqa: E402

GATING = {"softmax": Gating.SOFTMAX, "sigmoid_normalized": Gating.SIGMOID_NORMALIZED}

# (name, seed, E, k, d, f, B, gating)
FORWARD_CASES = [
    ("tiny_s0", 0, 4, 2, 8, 12, 9, "softmax"),
    ("tiny_s1", 1, 4, 2, 8, 12, 9, "sigmoid_normalized"),
    ("tiny_k1", 2, 3, 1, 5, 7, 6, "softmax"),
    ("tiny_k3", 3, 8, 3, 16, 24, 12, "softmax"),
    ("tiny_sig_k3", 4, 8, 3, 16, 24, 12, "sigmoid_normalized"),
    ("e1", 5, 1, 1, 8, 8, 4, "softmax"),
    ("b0", 6, 4, 2, 8, 12, 0, "softmax"),
    ("mid_e16_k4_sig", 7, 16, 4, 128, 192, 40, "sigmoid_normalized"),
    ("mid_e60_k4", 8, 60, 4, 64, 128, 48, "softmax"),
    ("small_s0", 0, 8, 2, 512, 1024, 128, "softmax"),
    ("small_s1", 1, 8, 2, 512, 1024, 128, "softmax"),
]

# (name, seed, B, d, E, k, gating, scaled, bf16_tokens)
ROUTE_CASES = [
    ("mixtral_b128", 11, 128, 4096, 8, 2, "softmax", True, True),
    ("mixtral_unscaled_b64", 12, 64, 4096, 8, 2, "softmax", False, False),
    ("qwen60_b128", 13, 128, 2048, 60, 4, "softmax", True, True),
    ("deepseek_b32", 14, 32, 7168, 256, 8, "sigmoid_normalized", True, True),
    ("deepseek_unscaled_b16", 15, 16, 7168, 256, 8, "sigmoid_normalized", False, False),
    ("skew64_b64", 16, 64, 3584, 64, 2, "softmax", True, True),
]


def forward_case(seed, e, k, d, f, b, gating):
    cfg = ModelConfig(e, k, d, f, GATING[gating])
    tokens, wr, gate, up, down = make_instance(seed, e, k, d, f, b)
    w = ExpertWeights(gate=gate, up=up, down=down)
    y, trace = moe_forward(tokens, wr, w, cfg, PipelineParams())
    routing = route(tokens, wr, cfg)
    counts = expert_histogram(routing, e)
    perm = build_permutation(routing)
    out = dict(
        y=y, indices=routing.indices, weights=routing.weights, counts=counts,
        forward=perm.forward, inverse=perm.inverse,
        trace_flops=np.array([r.flops for r in trace.records], dtype=np.int64),
        trace_bytes=np.array([r.total_bytes for r in trace.records], dtype=np.int64),
        trace_tiles=np.array([r.tiles for r in trace.records], dtype=np.int64),
    )
    if b <= 48:
        out["y_dense"] = dense_moe_oracle(tokens, wr, w, cfg)
    return out


def route_case(seed, b, d, e, k, gating, scaled, bf16):
    cfg = ModelConfig(e, k, d, 8, GATING[gating])
    tokens, wr = make_router_instance(seed, b, d, e, scaled=scaled, bf16_tokens=bf16)
    routing = route(tokens, wr, cfg)
    counts = expert_histogram(routing, e)
    perm = build_permutation(routing)
    logits = moeperf.linalg.dense_matmul(tokens, wr)
    return dict(indices=routing.indices, weights=routing.weights, counts=counts,
                forward=perm.forward, inverse=perm.inverse, logits=logits)


def topk_cases():
    """Tie-heavy score matrices through the reference ``topk_select``."""
    gen = np.random.Generator(np.random.PCG64(99))
    out = {}
    for name, e, k in (("e8k2", 8, 2), ("e60k4", 60, 4), ("e64k2", 64, 2), ("e256k8", 256, 8)):
        rows = []
        rows.append(np.zeros((4, e)))
        rows.append(np.round(gen.standard_normal((60, e)) * 2) / 4)  # many exact ties
        z = gen.standard_normal((60, e))
        z[gen.random((60, e)) < 0.6] = 0.0  # zero-heavy
        rows.append(np.abs(z))
        s = np.concatenate(rows).astype(np.float32)
        s = np.abs(s)
        for gname, g in GATING.items():
            r = topk_select(s, k, g)
            out[f"{name}_{gname}_scores"] = s
            out[f"{name}_{gname}_indices"] = r.indices
            out[f"{name}_{gname}_weights"] = r.weights
    return out


def main():
    meta = []
    arrays = {}
    for name, seed, e, k, d, f, b, g in FORWARD_CASES:
        res = forward_case(seed, e, k, d, f, b, g)
        for key, val in res.items():
            arrays[f"fwd/{name}/{key}"] = val
        meta.append(("fwd", name, seed, e, k, d, f, b, g))
        print("forward", name, flush=True)
    for name, seed, b, d, e, k, g, scaled, bf16 in ROUTE_CASES:
        res = route_case(seed, b, d, e, k, g, scaled, bf16)
        for key, val in res.items():
            arrays[f"route/{name}/{key}"] = val
        meta.append(("route", name, seed, e, k, d, int(scaled), b, g, int(bf16)))
        print("route", name, flush=True)
    for key, val in topk_cases().items():
        arrays[f"topk/{key}"] = val
    arrays["meta"] = np.array([repr(m) for m in meta])
    arrays["reference_version"] = np.array(moeperf.__version__)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
