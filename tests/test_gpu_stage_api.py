"""The reference's stage-level API on the GPU (paper_2605_23911_b200.stages).

The first half restates the reference's own router and scheduler tests
(/root/reference/pkg/tests/test_router.py, test_scheduler.py — same inputs,
same known answers, same exception classes) against this package's device
functions, and adds bit-for-bit comparisons with the oracle.  The second half
pushes the reference's edge cases through the FUSED CUDA router (the
identity-W_r trick: tokens are the logits, W_r = I, so x @ W_r is exact) and
checks the staged pipeline composition of pipeline.py:572-615.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import bits_equal  # noqa: E402
from oracle import moe_oracle as O  # noqa: E402

SOFTMAX_5000 = 0.9801866626534909  # reference tests/test_router.py:13
SOFTMAX_210M1 = [0.6439142598879722, 0.23688281808991013, 0.08714431874203257, 0.032058603280084995]


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2605_23911_b200 as pkg
    from paper_2605_23911_b200 import _lib
    _lib.load()
    return pkg


def _routing(P, indices):
    idx = np.asarray(indices, dtype=np.int64)
    return P.RoutingResult(indices=idx, weights=np.full(idx.shape, 0.5, dtype=np.float32))


# ---------------------------------------------------------------------------
# reference tests/test_router.py, restated against the device functions
# ---------------------------------------------------------------------------

def test_stable_softmax_row_frozen_values(P):  # test_router.py:22-31
    row = P.stable_softmax_row(np.array([5.0, 0.0, 0.0, 0.0]))
    assert np.isclose(float(row[0]), SOFTMAX_5000, rtol=1e-6)
    np.testing.assert_allclose(P.stable_softmax_row(np.array([2.0, 1.0, 0.0, -1.0])),
                               np.array(SOFTMAX_210M1, dtype=np.float32), rtol=1e-6)
    assert np.isclose(float(row.sum()), 1.0, atol=1e-6)
    bits_equal(row, O.gate_scores(np.array([[5.0, 0, 0, 0]], np.float32), "softmax")[0])


def test_softmax_large_magnitudes_finite(P):  # test_router.py:34-38
    scores = P.gate_scores(np.array([[1e4, -1e4, 0.0, 5.0]]), P.Gating.SOFTMAX)
    assert np.isfinite(scores).all()
    assert np.isclose(float(scores.sum()), 1.0, atol=1e-6)
    assert scores[0, 0] == np.float32(1.0)


def test_gate_scores_rejects_non_finite(P):  # test_router.py:41-45
    with pytest.raises(P.NonFiniteInput):
        P.gate_scores(np.array([[np.inf, 0.0]]), P.Gating.SOFTMAX)
    with pytest.raises(P.NonFiniteInput):
        P.gate_scores(np.array([[np.nan, 0.0]]), P.Gating.SIGMOID_NORMALIZED)


def test_topk_argmax_breaks_ties_toward_lowest_index(P):  # test_router.py:48-56
    r = P.topk_select(np.array([[0.25, 0.25, 0.25, 0.25]], dtype=np.float32), 2)
    assert r.indices.tolist() == [[0, 1]]
    r = P.topk_select(np.array([[0.0, 0.6, 0.0, 0.4]], dtype=np.float32), 3)
    assert r.indices.tolist() == [[1, 3, 0]]


def test_topk_never_reselects_even_zero_scores(P):  # test_router.py:59-63
    r = P.topk_select(np.zeros((3, 5), dtype=np.float32), 5)
    for row in r.indices:
        assert sorted(row.tolist()) == [0, 1, 2, 3, 4]


def test_topk_invalid_k(P):  # test_router.py:66-71
    scores = np.ones((2, 3), dtype=np.float32)
    with pytest.raises(P.InvalidK):
        P.topk_select(scores, 0)
    with pytest.raises(P.InvalidK):
        P.topk_select(scores, 4)


def test_sigmoid_normalized_weights_sum_to_one(P):  # test_router.py:74-78
    rng = np.random.Generator(np.random.PCG64(1234))
    logits = rng.standard_normal((32, 16)).astype(np.float32)
    scores = P.gate_scores(logits, P.Gating.SIGMOID_NORMALIZED)
    r = P.topk_select(scores, 4, P.Gating.SIGMOID_NORMALIZED)
    np.testing.assert_allclose(r.weights.sum(axis=1), 1.0, atol=1e-6)
    idx_ref, w_ref = O.topk_select(O.gate_scores(logits, "sigmoid_normalized"), 4, "sigmoid_normalized")
    bits_equal(r.indices, idx_ref)
    bits_equal(r.weights, w_ref)


def test_sigmoid_degenerate_row_falls_back_to_uniform(P):  # test_router.py:81-86
    logits = np.full((1, 4), -200.0, dtype=np.float32)
    scores = P.gate_scores(logits, P.Gating.SIGMOID_NORMALIZED)
    assert (scores == 0.0).all()
    r = P.topk_select(scores, 2, P.Gating.SIGMOID_NORMALIZED)
    assert (r.weights == np.float32(0.5)).all()


def test_route_single_dominant_logit(P):  # test_router.py:89-96
    cfg = P.ModelConfig(num_experts=4, top_k=1, hidden_dim=1, ffn_dim=4)
    r = P.route(np.array([[1.0]], np.float32), np.array([[5.0, 0.0, 0.0, 0.0]], np.float32), cfg)
    assert r.indices.tolist() == [[0]]
    assert np.isclose(float(r.weights[0, 0]), SOFTMAX_5000, rtol=1e-6)


def test_route_single_expert_weight_is_one(P):  # test_router.py:99-104
    cfg = P.ModelConfig(num_experts=1, top_k=1, hidden_dim=3, ffn_dim=4)
    r = P.route(np.array([[0.5, -1.0, 2.0]], np.float32), np.array([[1.0], [2.0], [3.0]], np.float32), cfg)
    assert r.weights[0, 0] == np.float32(1.0)


def test_route_zero_tokens(P):  # test_router.py:107-114
    cfg = P.ModelConfig(num_experts=4, top_k=2, hidden_dim=3, ffn_dim=4)
    r = P.route(np.zeros((0, 3), np.float32), np.zeros((3, 4), np.float32), cfg)
    assert r.indices.shape == (0, 2) and r.weights.shape == (0, 2)


def test_route_shape_errors(P):  # test_router.py:117-122
    cfg = P.ModelConfig(num_experts=4, top_k=2, hidden_dim=3, ffn_dim=4)
    with pytest.raises(P.ShapeMismatch):
        P.route(np.zeros((2, 5), np.float32), np.zeros((3, 4), np.float32), cfg)
    with pytest.raises(P.ShapeMismatch):
        P.route(np.zeros((2, 3), np.float32), np.zeros((3, 5), np.float32), cfg)


@pytest.mark.parametrize("seed", range(24))
def test_topk_properties_bitexact(P, seed):  # test_router.py:125-145 (+ bit-exact vs the oracle)
    rng = np.random.default_rng(seed)
    E = int(rng.integers(1, 13))
    k = min(int(rng.integers(1, 7)), E)
    B = int(rng.integers(0, 17))
    gating = ["softmax", "sigmoid_normalized"][seed % 2]
    logits = np.random.Generator(np.random.PCG64(seed)).standard_normal((B, E)).astype(np.float32)
    scores = P.gate_scores(logits, P.Gating(gating))
    r = P.topk_select(scores, k, P.Gating(gating))
    assert r.indices.shape == (B, k)
    for row in r.indices:
        assert len(set(row.tolist())) == k
    raw = scores[np.arange(B)[:, None], r.indices]
    assert (np.diff(raw, axis=1) <= 0).all()
    assert (r.weights >= 0).all()
    bits_equal(scores, O.gate_scores(logits, gating))
    idx_ref, w_ref = O.topk_select(O.gate_scores(logits, gating), k, gating)
    bits_equal(r.indices, idx_ref)
    bits_equal(r.weights, w_ref)


# ---------------------------------------------------------------------------
# reference tests/test_scheduler.py, restated
# ---------------------------------------------------------------------------

def test_offsets_and_schedule_worked_example(P):  # test_scheduler.py:24-36
    offsets = P.expert_offsets([5, 0, 7])
    assert offsets.offsets.tolist() == [0, 5, 5, 12]
    assert offsets.num_experts == 3 and offsets.total == 12 and offsets.count(1) == 0
    schedule = P.build_block_schedule(offsets, 4)
    assert schedule.entries == ((0, 0), (0, 4), (2, 0), (2, 4)) and len(schedule) == 4
    for bad in (0, -1, 2.5, True):  # test_scheduler.py:39-47
        with pytest.raises(P.InvalidBlockM):
            P.build_block_schedule(P.expert_offsets([3, 2]), bad)


def test_histogram_counts_and_validation(P):  # test_scheduler.py:50-57
    counts = P.expert_histogram(_routing(P, [[1, 0], [0, 1], [0, 0]]), 3)
    assert counts.tolist() == [4, 2, 0] and counts.dtype == np.int64
    with pytest.raises(P.IndexOutOfRange):
        P.expert_histogram(_routing(P, [[0, 5]]), 3)
    with pytest.raises(P.IndexOutOfRange):
        P.expert_histogram(_routing(P, [[-1, 0]]), 3)
    with pytest.raises(P.IndexOutOfRange):  # test_scheduler.py:60-64
        P.expert_offsets([2, -1])
    with pytest.raises(P.ShapeMismatch):
        P.expert_offsets(np.zeros((2, 2), dtype=np.int64))


def test_permutation_stable_within_expert(P):  # test_scheduler.py:67-74
    perm = P.build_permutation(_routing(P, [[1, 0], [0, 1], [0, 0]]))
    assert perm.forward.tolist() == [1, 2, 4, 5, 0, 3]
    assert perm.inverse[perm.forward].tolist() == list(range(6))
    assert perm.forward[perm.inverse].tolist() == list(range(6))


def test_empty_routing_permutation_and_schedule(P):  # test_scheduler.py:77-86
    r = P.RoutingResult(indices=np.zeros((0, 2), np.int64), weights=np.zeros((0, 2), np.float32))
    assert P.build_permutation(r).forward.size == 0
    schedule = P.build_block_schedule(P.expert_offsets(P.expert_histogram(r, 4)), 8)
    assert schedule.entries == ()


@pytest.mark.parametrize("seed", range(16))
def test_permutation_is_expert_major_and_stable(P, seed):  # test_scheduler.py:110-129 (+ vs the oracle)
    rng = np.random.default_rng(1000 + seed)
    E = int(rng.integers(1, 11))
    k = min(int(rng.integers(1, 6)), E)
    B = int(rng.integers(0, 41)) if seed else 40
    gen = np.random.Generator(np.random.PCG64(seed))
    idx = np.empty((B, k), dtype=np.int64)
    for t in range(B):
        idx[t] = gen.choice(E, size=k, replace=False)
    r = P.RoutingResult(indices=idx, weights=np.ones((B, k), np.float32))
    perm = P.build_permutation(r)
    flat = idx.reshape(-1)
    srt = flat[perm.forward]
    assert (np.diff(srt) >= 0).all()
    for e in range(E):
        assert (np.diff(perm.forward[srt == e]) > 0).all()
    assert np.array_equal(perm.inverse[perm.forward], np.arange(B * k))
    fwd_ref, inv_ref = O.build_permutation(idx)
    bits_equal(perm.forward, fwd_ref)
    bits_equal(perm.inverse, inv_ref)
    bits_equal(P.expert_histogram(r, E), O.expert_histogram(idx, E))


# ---------------------------------------------------------------------------
# the staged pipeline (pipeline.py:572-615) through the stage API
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("case", [(0, 8, 2, 512, 1024, 128, "softmax"), (3, 16, 4, 96, 200, 37, "sigmoid_normalized"),
                                  (5, 4, 2, 8, 12, 9, "softmax")])
def test_staged_pipeline_against_oracle(P, case):
    seed, e, k, d, f, b, g = case
    tokens, wr, gate, up, down = O.make_instance(seed, e, k, d, f, b)
    cfg = P.ModelConfig(e, k, d, f, P.Gating(g))
    params = P.PipelineParams()
    ref = O.moe_forward(tokens, wr, gate, up, down, e, k, g)
    routing = P.route(tokens, wr, cfg)
    bits_equal(routing.indices, ref["indices"])
    bits_equal(routing.weights, ref["weights"])
    counts = P.expert_histogram(routing, e)
    bits_equal(counts, ref["counts"])
    offsets = P.expert_offsets(counts)
    perm = P.build_permutation(routing)
    bits_equal(perm.forward, ref["forward"])
    schedule = P.build_block_schedule(offsets, params.block_m)
    xp = P.permute_tokens(tokens, routing, perm)
    bits_equal(xp, ref["permuted"])  # exact fp32 gather
    w = P.ExpertWeights(gate, up, down)
    tr = P.PipelineTrace(element_bytes=4)
    h = P.fused_gate_up(xp, w, schedule, offsets, params, tr)
    h_u = P.unfused_gate_up(xp, w, schedule, offsets, params)
    bits_equal(h_u, h)  # the reference's fused == unfused invariant
    assert O.max_rel_error(h, ref["h"]) < 1e-2
    ys = P.grouped_gemm(h, down, schedule, offsets, params, tr)
    assert O.max_rel_error(ys, ref["expert_out"]) < 2e-2
    # the combine is exact: fed the oracle's expert outputs it reproduces y bit for bit
    bits_equal(P.unpermute_combine(ref["expert_out"], routing, perm), ref["y"])
    y = P.unpermute_combine(ys, routing, perm)
    assert O.max_rel_error(y, ref["y"]) <= 2e-2
    assert [r.stage for r in tr.records] == ["GateUp", "Down"]
    full = P.trace_from_counts(cfg, b, counts, params)
    assert tr.records[0].flops == full.stage("GateUp").flops and tr.records[1].flops == full.stage("Down").flops
    assert tr.records[0].total_bytes == full.stage("GateUp").total_bytes * 4 // full.element_bytes


def test_stage_errors_match_reference(P):
    tokens, wr, gate, up, down = O.make_instance(1, 4, 2, 8, 12, 9)
    cfg = P.ModelConfig(4, 2, 8, 12)
    routing = P.route(tokens, wr, cfg)
    perm = P.build_permutation(routing)
    offsets = P.expert_offsets(P.expert_histogram(routing, 4))
    with pytest.raises(P.ShapeMismatch):
        P.permute_tokens(tokens[:5], routing, perm)
    with pytest.raises(P.ShapeMismatch):
        P.unpermute_combine(np.zeros((5, 8), np.float32), routing, perm)
    bad = P.BlockSchedule(entries=((0, 0),), block_m=64)
    with pytest.raises(P.ScheduleMismatch):
        P.grouped_gemm(np.zeros((18, 12), np.float32), down, bad, offsets, P.PipelineParams())
    with pytest.raises(P.ShapeMismatch):
        P.fused_gate_up(np.zeros((18, 8), np.float32), P.ExpertWeights(gate, up[:8], down),
                        P.build_block_schedule(offsets, 64), offsets, P.PipelineParams())


def test_numerics_helpers_bitexact(P):
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.standard_normal(99995) * 30, [0.0, -0.0, 1e4, -1e4, 88.7, -103.9, -104.0]]).astype(
        np.float32).reshape(-1, 7)
    bits_equal(P.sigmoid(x), O.sigmoid_f32(x))
    bits_equal(P.silu(x), O.silu_f32(x))
    assert float(P.sigmoid(np.zeros(1, np.float32))[0]) == 0.5  # test_linalg.py:70-83
    assert np.isclose(float(P.silu(np.ones(1, np.float32))[0]), 0.7310585786300049, rtol=1e-6)
    a = rng.standard_normal((37, 300)).astype(np.float32)
    b = rng.standard_normal((300, 19)).astype(np.float32)
    bits_equal(P.dense_matmul(a, b), O.dot_fp64_fold(a, b))
    with pytest.raises(P.ShapeMismatch):
        P.dense_matmul(a, b[:5])


def test_sigmoid_port_exhaustive(P):
    """The numpy-SIMD float32 exp port behind the router's sigmoid, over EVERY
    float32 in [-110, 110] (2 x 1.12e9 values), against this box's numpy
    (whose exp kernel is chosen per CPU at runtime): bit-for-bit."""
    lo_bits = np.uint32(0x80000000)  # -0.0
    hi_bits = np.uint32(0xC2DC0000)  # -110.0
    chunk = 1 << 27
    dev = torch.device("cuda")
    for sign_bits in (np.uint32(0), lo_bits):
        start, stop = 0, int(hi_bits - lo_bits) + 1
        for c0 in range(start, stop, chunk):
            n = min(chunk, stop - c0)
            bits = (np.arange(c0, c0 + n, dtype=np.uint32) | sign_bits)
            x = bits.view(np.float32)
            xt = torch.from_numpy(x).to(dev)
            y = P.sigmoid(xt).cpu().numpy()
            ref = O.sigmoid_f32(x)
            if not np.array_equal(y.view(np.uint32), ref.view(np.uint32)):
                bad = np.nonzero(y.view(np.uint32) != ref.view(np.uint32))[0]
                raise AssertionError(f"{bad.size} mismatches, first x={x[bad[0]]!r} got {y[bad[0]]!r} "
                                     f"want {ref[bad[0]]!r}")


def test_softmax_exp_port_exhaustive(P):
    """The softmax's float64 exp (router.cuh np_exp64, the port of numpy's
    SVML exp) against THIS box's np.exp on every float32 input the softmax
    can feed it (s = fp32(l - max) in (-707.70, 0]; 1.13e9 values), bit for
    bit.  (numpy picks its exp kernel per CPU at run time: the check runs
    where the parity is claimed.)"""
    from paper_2605_23911_b200 import _lib
    lib = _lib.load()
    hi = int(np.array([-707.70327], np.float32).view(np.uint32)[0])
    chunk = 1 << 26
    dev = torch.device("cuda")
    total = 0
    for c0 in range(0x80000000, hi + 1, chunk):
        c1 = min(hi + 1, c0 + chunk)
        x = np.arange(c0, c1, dtype=np.uint64).astype(np.uint32).view(np.float32).astype(np.float64)
        x = x[np.abs(x) < 707.7032713517042]
        xt = torch.from_numpy(x).to(dev)
        yt = torch.empty_like(xt)
        _lib.check(lib.moe_b200_np_exp64(x.size, xt.data_ptr(), yt.data_ptr(), torch.cuda.current_stream().cuda_stream),
                   "np_exp64")
        y = yt.cpu().numpy()
        ref = np.exp(x)
        if not np.array_equal(y.view(np.uint64), ref.view(np.uint64)):
            bad = np.nonzero(y.view(np.uint64) != ref.view(np.uint64))[0]
            raise AssertionError(f"{bad.size} mismatches, first x={x[bad[0]]!r}: {y[bad[0]]!r} vs {ref[bad[0]]!r}")
        total += x.size
    assert total > 1_100_000_000


# ---------------------------------------------------------------------------
# the reference's edge cases through the FUSED router kernels (identity W_r)
# ---------------------------------------------------------------------------

ROUTER_MODES = {
    "auto": {},
    "fallback": {"MOE_B200_ROUTER_FORCE_EXACT": "1"},
    "exact_kernel": {"MOE_B200_SEG_MAX_CHAINS": "0"},
}


def _identity_layer(P, E, k, gating, B):
    z = np.zeros((E * E, 8), np.float32)
    cfg = P.ModelConfig(E, k, E, 8, P.Gating(gating))
    return P.MoELayer(cfg, P.ExpertWeights(z, z, np.zeros((E * 8, E), np.float32)), np.eye(E, dtype=np.float32),
                      max_tokens=B)


def _route_logits(P, logits, k, gating):
    B, E = logits.shape
    layer = _identity_layer(P, E, k, gating, B)
    r = layer.route(torch.from_numpy(np.ascontiguousarray(logits)).cuda(), logits=True)
    torch.cuda.synchronize()
    out = {n: r[n].cpu().numpy() for n in ("indices", "weights", "logits", "counts", "forward")}
    out["flags"] = layer.read_flags()
    return out


@pytest.mark.parametrize("mode", sorted(ROUTER_MODES))
def test_fused_router_reference_edge_cases(P, mode, monkeypatch):
    """test_router.py:48-86 ties / never reselecting / -200 zero-sum fallback,
    as logits through the fused router: indices and weights bit-exact."""
    for k_, v_ in ROUTER_MODES[mode].items():
        monkeypatch.setenv(k_, v_)
    cases = [
        (np.zeros((3, 4), np.float32), 2, "softmax"),                     # all-equal scores -> [0, 1]
        (np.array([[0.0, 3.0, 0.0, 2.0]] * 2, np.float32), 3, "softmax"),  # zero-heavy ties
        (np.zeros((3, 5), np.float32), 5, "sigmoid_normalized"),           # never reselect
        (np.full((2, 4), -200.0, np.float32), 2, "sigmoid_normalized"),    # zero-sum fallback -> 1/k
        (np.full((2, 8), -200.0, np.float32), 8, "sigmoid_normalized"),    # k = 8 pairwise order
        (np.array([[1e4, -1e4, 0.0, 5.0]], np.float32), 2, "softmax"),     # saturation
    ]
    for logits, k, g in cases:
        got = _route_logits(P, logits, k, g)
        idx_ref, w_ref = O.route(logits, np.eye(logits.shape[1], dtype=np.float32), k, g)
        bits_equal(got["logits"], logits)
        bits_equal(got["indices"].astype(np.int64), idx_ref)
        bits_equal(got["weights"], w_ref)
        assert got["flags"] == 0
    assert _route_logits(P, np.full((2, 4), -200.0, np.float32), 2, "sigmoid_normalized")["weights"].tolist() == \
        [[0.5, 0.5], [0.5, 0.5]]


@pytest.mark.parametrize("mode", ["auto", "exact_kernel"])
def test_c10_router_robustness_at_scale(P, mode, monkeypatch):
    """test_acceptance.py:350-384 (C10): 1e5 x 256 logits x1e4 with zero rows:
    through the stage API AND the fused router, bit-exact with the oracle; the
    zero rows route to experts 0..7."""
    for k_, v_ in ROUTER_MODES[mode].items():
        monkeypatch.setenv(k_, v_)
    gen = np.random.Generator(np.random.PCG64(99))
    rows, E = 100_000, 256
    logits = (gen.standard_normal((rows, E)) * 1e4).astype(np.float32)
    logits[: rows // 10] = 0.0
    scores_ref = O.gate_scores(logits, "softmax")
    idx_ref, w_ref = O.topk_select(scores_ref, 8, "softmax")
    if mode == "auto":
        scores = P.gate_scores(logits, P.Gating.SOFTMAX)
        bits_equal(scores, scores_ref)
        r = P.topk_select(scores, 8, P.Gating.SOFTMAX)
        bits_equal(r.indices, idx_ref)
        bits_equal(r.weights, w_ref)
        with pytest.raises(P.InvalidK):
            P.topk_select(scores[:4], 257, P.Gating.SOFTMAX)
    # the fused router on the first 20k rows (all 10k zero rows included)
    n = 20_000
    got = _route_logits(P, logits[:n], 8, "softmax")
    bits_equal(got["indices"].astype(np.int64), idx_ref[:n])
    bits_equal(got["weights"], w_ref[:n])
    assert (got["indices"][: rows // 10] == np.arange(8)).all()
    bits_equal(got["counts"].astype(np.int64), O.expert_histogram(idx_ref[:n], E))
    bits_equal(got["forward"].astype(np.int64), O.build_permutation(idx_ref[:n])[0])


@pytest.mark.parametrize("gating", ["softmax", "sigmoid_normalized"])
def test_certificate_recompute_fires_near_midpoints(P, gating):
    """Logits whose exact fp64 fold sits one fp64 ulp above or below an fp32
    rounding midpoint: the segment router's certified interval straddles the
    midpoint, phase 2 must recompute them with the exact chain, and the
    routing must still be bit-exact (the recompute count is read back through
    the router's debug counters)."""
    from paper_2605_23911_b200 import _lib
    lib = _lib.load()
    E, k, d, B = 8, 2, 64, 64
    rng = np.random.default_rng(5)
    a = (rng.uniform(1.0, 2.0, E) * rng.choice([-1.0, 1.0], E)).astype(np.float32)
    half_ulp = (np.spacing(np.abs(a)) / 2).astype(np.float32) * np.sign(a).astype(np.float32)
    wr = np.zeros((d, E), np.float32)
    wr[0] = a
    wr[1] = half_ulp
    wr[2] = np.float32(2.0 ** -52)
    wr[3:] = (rng.standard_normal((d - 3, E)) * 1e-30).astype(np.float32)  # long chain, negligible mass
    x = np.zeros((B, d), np.float32)
    x[:, 0] = 1.0
    x[:, 1] = 1.0
    x[:, 2] = rng.choice([-1.0, 1.0], B).astype(np.float32)  # above / below the midpoint per token
    cfg = P.ModelConfig(E, k, d, 8, P.Gating(gating))
    z = np.zeros((E * d, 8), np.float32)
    layer = P.MoELayer(cfg, P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
    trace = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    lib.moe_b200_debug_set_router_trace.argtypes = [ctypes.c_void_p]
    lib.moe_b200_debug_set_router_trace(ctypes.c_void_p(trace.data_ptr()))
    try:
        r = layer.route(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
    finally:
        lib.moe_b200_debug_set_router_trace(ctypes.c_void_p(0))
    recomputed = int(trace.view(-1, 16)[:, 11:13].sum())
    idx_ref, w_ref = O.route(x, wr, k, gating)
    bits_equal(r["indices"].cpu().numpy().astype(np.int64), idx_ref)
    bits_equal(r["weights"].cpu().numpy(), w_ref)
    # the midpoint construction really is ambiguous: both roundings occur
    lg = O.router_logits(x, wr)
    assert (lg != a[None, :]).any() and (lg == a[None, :]).any()
    assert recomputed > 0, "the certificate never sent a logit to the exact chain"


def test_certificate_enumeration_avoids_recompute(P):
    """Softmax routing with ONE logit (a non-selected expert, far below the
    row max) whose exact fold sits one fp64 ulp from an fp32 rounding
    midpoint: its certified interval holds two fp32 candidates, and phase 2
    evaluates the token's outputs for both instead of running the exact chain.
    Routing stays bit-exact, the enumeration fires and no logit is recomputed."""
    from paper_2605_23911_b200 import _lib
    lib = _lib.load()
    E, k, d, B = 8, 2, 64, 64
    rng = np.random.default_rng(11)
    a = np.array([2.0, 1.75, 0.5, -0.25, 1.0, -1.0, 0.125, -20.3], np.float32)
    wr = np.zeros((d, E), np.float32)
    wr[0] = a
    wr[1, 7] = np.float32(np.spacing(np.float32(20.3)) / 2) * -1.0   # half an fp32 ulp (toward -inf)
    wr[2, 7] = np.float32(2.0 ** -48)                                 # one fp64 ulp at |l| ~ 20
    wr[3:] = (rng.standard_normal((d - 3, E)) * 1e-30).astype(np.float32)
    x = np.zeros((B, d), np.float32)
    x[:, 0] = 1.0
    x[:, 1] = 1.0
    x[:, 2] = rng.choice([-1.0, 1.0], B).astype(np.float32)
    cfg = P.ModelConfig(E, k, d, 8, P.Gating("softmax"))
    z = np.zeros((E * d, 8), np.float32)
    layer = P.MoELayer(cfg, P.ExpertWeights(z, z, np.zeros((E * 8, d), np.float32)), wr, max_tokens=B)
    trace = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
    lib.moe_b200_debug_set_router_trace.argtypes = [ctypes.c_void_p]
    lib.moe_b200_debug_set_router_trace(ctypes.c_void_p(trace.data_ptr()))
    try:
        r = layer.route(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
    finally:
        lib.moe_b200_debug_set_router_trace(ctypes.c_void_p(0))
    t = trace.view(-1, 16).cpu().numpy()
    enumerated = int((t[:, 12] >> 32).sum())
    recomputed = int(t[:, 11].sum() + (t[:, 12] & 0xFFFFFFFF).sum())
    idx_ref, w_ref = O.route(x, wr, k, "softmax")
    bits_equal(r["indices"].cpu().numpy().astype(np.int64), idx_ref)
    bits_equal(r["weights"].cpu().numpy(), w_ref)
    lg = O.router_logits(x, wr)
    assert len(np.unique(lg[:, 7])) == 2, "the construction should put expert 7 on both sides of the midpoint"
    assert enumerated > 0, "the enumeration certificate never fired"
    assert recomputed == 0, f"{recomputed} logits went to the exact chain"
