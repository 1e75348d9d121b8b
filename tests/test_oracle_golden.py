"""Pin the CPU oracle against the reference's own outputs (golden fixtures)
and the known answers the reference's tests hold."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import moe_oracle as O
from golden_util import bits_equal as _bits_equal, golden_meta


def _forward_cases(golden):
    return [m for m in golden_meta(golden) if m[0] == "fwd"]


def _route_cases(golden):
    return [m for m in golden_meta(golden) if m[0] == "route"]


def test_oracle_forward_matches_reference_bitwise(golden):
    cases = _forward_cases(golden)
    assert len(cases) >= 10
    for _, name, seed, e, k, d, f, b, g in cases:
        tokens, wr, gate, up, down = O.make_instance(seed, e, k, d, f, b)
        res = O.moe_forward(tokens, wr, gate, up, down, e, k, g)
        p = f"fwd/{name}/"
        _bits_equal(res["indices"], golden[p + "indices"])
        _bits_equal(res["weights"], golden[p + "weights"])
        _bits_equal(res["counts"], golden[p + "counts"])
        _bits_equal(res["forward"], golden[p + "forward"])
        _bits_equal(res["inverse"], golden[p + "inverse"])
        _bits_equal(res["y"], golden[p + "y"])
        if p + "y_dense" in golden:
            yd = O.dense_moe_oracle(tokens, wr, gate, up, down, e, k, g)
            _bits_equal(yd, golden[p + "y_dense"])


def test_oracle_route_full_shapes_bitwise(golden):
    for _, name, seed, e, k, d, scaled, b, g, bf16 in _route_cases(golden):
        tokens, wr = O.make_router_instance(seed, b, d, e, scaled=bool(scaled), bf16_tokens=bool(bf16))
        p = f"route/{name}/"
        logits = O.router_logits(tokens, wr)
        _bits_equal(logits, golden[p + "logits"])
        idx, w = O.topk_select(O.gate_scores(logits, g), k, g)
        _bits_equal(idx, golden[p + "indices"])
        _bits_equal(w, golden[p + "weights"])
        _bits_equal(O.expert_histogram(idx, e), golden[p + "counts"])
        fwd, inv = O.build_permutation(idx)
        _bits_equal(fwd, golden[p + "forward"])
        _bits_equal(inv, golden[p + "inverse"])


def test_oracle_topk_tie_heavy_bitwise(golden):
    names = sorted({k.rsplit("_", 1)[0] for k in golden if k.startswith("topk/")})
    assert names
    for base in names:
        scores = golden[base + "_scores"]
        gating = "sigmoid_normalized" if "sigmoid" in base else "softmax"
        k = int(base.split("k")[-1].split("_")[0])
        idx, w = O.topk_select(scores, k, gating)
        _bits_equal(idx, golden[base + "_indices"])
        _bits_equal(w, golden[base + "_weights"])


# ---- known answers held by the reference's own tests --------------------------------

def test_known_softmax_values():
    # tests/test_router.py:13-31
    s = O.gate_scores(np.array([[5.0, 0, 0, 0], [2.0, 1.0, 0.0, -1.0]], dtype=np.float32), O.SOFTMAX)
    assert np.isclose(float(s[0, 0]), 0.9801866626534909, rtol=1e-6)
    np.testing.assert_allclose(s[1], [0.6439142598879722, 0.23688281808991013,
                                      0.08714431874203257, 0.032058603280084995], rtol=1e-6)
    big = O.gate_scores(np.array([[1e4, -1e4, 0.0, 5.0]], dtype=np.float32), O.SOFTMAX)
    assert big[0, 0] == np.float32(1.0)


def test_known_topk_ties():
    # tests/test_router.py:48-62
    idx, _ = O.topk_select(np.full((1, 4), 0.25, np.float32), 2, O.SOFTMAX)
    assert idx.tolist() == [[0, 1]]
    idx, _ = O.topk_select(np.array([[0.0, 0.6, 0.0, 0.4]], np.float32), 3, O.SOFTMAX)
    assert idx.tolist() == [[1, 3, 0]]
    idx, _ = O.topk_select(np.zeros((3, 5), np.float32), 5, O.SOFTMAX)
    for row in idx:
        assert sorted(row.tolist()) == [0, 1, 2, 3, 4]


def test_known_sigmoid_fallback_and_single_expert():
    # tests/test_router.py:80-104
    s = O.gate_scores(np.full((1, 4), -200.0, np.float32), O.SIGMOID_NORMALIZED)
    assert (s == 0).all()
    _, w = O.topk_select(s, 2, O.SIGMOID_NORMALIZED)
    assert (w == np.float32(0.5)).all()
    idx, w = O.route(np.array([[1.0]], np.float32), np.array([[5.0, 0, 0, 0]], np.float32), 1, O.SOFTMAX)
    assert idx.tolist() == [[0]] and np.isclose(float(w[0, 0]), 0.9801866626534909, rtol=1e-6)
    _, w = O.route(np.array([[0.5, -1.0, 2.0]], np.float32), np.array([[1.0], [2.0], [3.0]], np.float32), 1, O.SOFTMAX)
    assert w[0, 0] == np.float32(1.0)


def test_known_scheduler_examples():
    # tests/test_scheduler.py:24-74
    off = O.expert_offsets(np.array([5, 0, 7]))
    assert off.tolist() == [0, 5, 5, 12]
    assert O.build_block_schedule(off, 4) == ((0, 0), (0, 4), (2, 0), (2, 4))
    idx = np.array([[1, 0], [0, 1], [0, 0]])
    assert O.expert_histogram(idx, 3).tolist() == [4, 2, 0]
    fwd, inv = O.build_permutation(idx)
    assert fwd.tolist() == [1, 2, 4, 5, 0, 3]
    assert inv[fwd].tolist() == list(range(6))


def test_known_silu_and_sigmoid():
    # tests/test_linalg.py:70-83
    assert O.sigmoid_f32(np.float32(0.0)) == np.float32(0.5)
    assert np.isclose(float(O.silu_f32(np.float32(1.0))), 0.7310585786300049, rtol=1e-6)
    s = O.sigmoid_f32(np.array([1e4, -1e4], np.float32))
    assert s[0] == 1.0 and s[1] == 0.0


def test_fold_order_is_scalar_definition():
    # tests/test_linalg.py:15-32: result equals the scalar left-to-right fold
    rng = np.random.default_rng(5)
    a = rng.standard_normal((3, 37)).astype(np.float32)
    b = rng.standard_normal((37, 4)).astype(np.float32)
    c = O.dot_fp64_fold(a, b)
    for i in range(3):
        for j in range(4):
            acc = float(a[i, 0]) * float(b[0, j])
            for kk in range(1, 37):
                acc = acc + float(a[i, kk]) * float(b[kk, j])
            assert np.float32(acc) == c[i, j]


def test_acceptance_c10_router_robustness():
    # tests/test_acceptance.py:350-384 (scaled down): huge logits, zero-heavy rows
    rng = np.random.default_rng(0)
    logits = (rng.standard_normal((2000, 256)) * 1e4).astype(np.float32)
    logits[::7] = 0.0
    for g in (O.SOFTMAX, O.SIGMOID_NORMALIZED):
        idx, w = O.topk_select(O.gate_scores(logits, g), 8, g)
        assert np.isfinite(w).all()
        assert (np.sort(idx[::7], axis=1) == np.arange(8)).all()
