"""GPU tests of the screening router (csrc/router_screen.cuh): INT8 tensor-core
screen + candidate refinement + certified phase 2 for sigmoid gating.

Every case routes through the C-ABI with MOE_B200_SCREEN=1 (the screen for any
sigmoid batch; by default it serves the exact router's regime, B x E > 64K)
and compares indices, weight bits, counts and the permutation with the oracle
(oracle/moe_oracle.py route: the reference's router.py:88-133 restated)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from golden_util import bits_equal  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2605_23911_b200 as pkg

    return pkg


def _route(P, x, wr, k, monkeypatch, screen="1"):
    e = wr.shape[1]
    d = wr.shape[0]
    monkeypatch.setenv("MOE_B200_SCREEN", screen)
    cfg = P.ModelConfig(e, k, d, 8, P.Gating("sigmoid_normalized"))
    z = np.zeros((e * d, 8), np.float32)
    layer = P.MoELayer(cfg, P.ExpertWeights(z, z, np.zeros((e * 8, d), np.float32)), wr, max_tokens=x.shape[0])
    r = layer.route(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    assert layer.read_flags() == 0
    return {kk: v.cpu().numpy() for kk, v in r.items() if v is not None}


def _check(P, x, wr, k, monkeypatch):
    r = _route(P, x, wr, k, monkeypatch)
    idx_ref, w_ref = O.route(x, wr, k, "sigmoid_normalized")
    bits_equal(r["indices"].astype(np.int64), idx_ref)
    bits_equal(r["weights"], w_ref)
    counts = np.bincount(idx_ref.reshape(-1), minlength=wr.shape[1])
    bits_equal(r["counts"].astype(np.int64), counts)
    fwd_ref = np.argsort(idx_ref.reshape(-1), kind="stable")
    bits_equal(r["forward"].astype(np.int64), fwd_ref)


@pytest.mark.parametrize("shape", [
    (512, 7168, 256, 8),   # DeepSeek-V3 (the benched config)
    (37, 1000, 256, 8),    # ragged B and d
    (300, 300, 200, 6),    # E not a multiple of the 128-expert tile
    (1, 128, 32, 2),
    (130, 96, 64, 4),
])
def test_screen_router_bitexact(P, shape, monkeypatch):
    b, d, e, k = shape
    rng = np.random.default_rng(b * 7 + d)
    x = rng.standard_normal((b, d)).astype(np.float32)
    wr = (rng.standard_normal((d, e)) / np.sqrt(d)).astype(np.float32)
    _check(P, x, wr, k, monkeypatch)


def test_screen_router_ties_and_zero_rows(P, monkeypatch):
    """Duplicated expert columns (equal logits: ties broken toward the lowest
    index), zero token rows (every score 0.5), a row of huge range (tiny and
    large entries: digits far below the row maximum)."""
    rng = np.random.default_rng(5)
    b, d, e, k = 200, 512, 128, 8
    x = rng.standard_normal((b, d)).astype(np.float32)
    wr = (rng.standard_normal((d, e)) / np.sqrt(d)).astype(np.float32)
    wr[:, 10] = wr[:, 3]
    wr[:, 77] = wr[:, 3]
    wr[:, 100] = wr[:, 50]
    x[7] = 0.0
    x[8, :] = 0.0
    x[8, 5] = 1.0e-30
    x[9] *= np.float32(1e-6)
    x[9, 0] = 1.0e3
    x[10] = np.where(rng.random(d) < 0.5, 1e-38, 3e4).astype(np.float32)
    _check(P, x, wr, k, monkeypatch)


def test_screen_router_saturated_scores(P, monkeypatch):
    """Huge logits: most sigmoid scores are exactly 1.0 (ties across many
    experts), tokens with more than 32 candidates take the exact fallback."""
    rng = np.random.default_rng(11)
    b, d, e, k = 64, 256, 96, 4
    x = rng.standard_normal((b, d)).astype(np.float32)
    wr = (rng.standard_normal((d, e)) * 30.0).astype(np.float32)
    _check(P, x, wr, k, monkeypatch)


def test_screen_router_bf16_tokens(P, monkeypatch):
    rng = np.random.default_rng(3)
    b, d, e, k = 160, 640, 256, 8
    x32 = torch.from_numpy(rng.standard_normal((b, d)).astype(np.float32)).to(torch.bfloat16)
    wr = (rng.standard_normal((d, e)) / np.sqrt(d)).astype(np.float32)
    monkeypatch.setenv("MOE_B200_SCREEN", "1")
    cfg = P.ModelConfig(e, k, d, 8, P.Gating("sigmoid_normalized"))
    z = np.zeros((e * d, 8), np.float32)
    layer = P.MoELayer(cfg, P.ExpertWeights(z, z, np.zeros((e * 8, d), np.float32)), wr, max_tokens=b)
    r = layer.route(x32.cuda())
    idx_ref, w_ref = O.route(x32.float().numpy(), wr, k, "sigmoid_normalized")
    bits_equal(r["indices"].cpu().numpy().astype(np.int64), idx_ref)
    bits_equal(r["weights"].cpu().numpy(), w_ref)


def test_screen_router_matches_exact_router_on_layer(P, monkeypatch):
    """The DeepSeek-V3 layer forward with the screen (default at 512 tokens)
    and with the exact router (MOE_B200_SCREEN=0): identical routing and y."""
    rng = np.random.default_rng(17)
    e, k, d, f, b = 256, 8, 7168, 256, 512
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((b, d), generator=gen, device="cuda")
    wr = (torch.randn((d, e), generator=gen, device="cuda") / d ** 0.5).float()
    gate = (torch.randn((e * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    up = (torch.randn((e * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    down = (torch.randn((e * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
    outs = []
    for mode in ("-1", "0"):
        monkeypatch.setenv("MOE_B200_SCREEN", mode)
        cfg = P.ModelConfig(e, k, d, f, P.Gating("sigmoid_normalized"))
        layer = P.MoELayer(cfg, P.ExpertWeights(gate, up, down), wr, max_tokens=b)
        y = layer.forward(x)
        torch.cuda.synchronize()
        outs.append((y.cpu(), layer.topk_idx[:b].cpu(), layer.topk_w[:b].cpu()))
        del layer
    assert torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][2].view(torch.int32), outs[1][2].view(torch.int32))
    assert torch.equal(outs[0][0].view(torch.int32), outs[1][0].view(torch.int32))
    del rng


def test_screen_router_max_experts_and_k(P, monkeypatch):
    """E = 1024 (the library maximum: 8 expert tiles) and k = 32 (the
    candidate-list capacity; any tie or near-tie spills into the exact
    fallback), 150 tokens: the default regime (B x E > 64K chains)."""
    rng = np.random.default_rng(21)
    b, d, e, k = 150, 384, 1024, 32
    x = rng.standard_normal((b, d)).astype(np.float32)
    wr = (rng.standard_normal((d, e)) / np.sqrt(d)).astype(np.float32)
    r = _route(P, x, wr, k, monkeypatch, screen="-1")
    idx_ref, w_ref = O.route(x, wr, k, "sigmoid_normalized")
    bits_equal(r["indices"].astype(np.int64), idx_ref)
    bits_equal(r["weights"], w_ref)


def test_screen_router_inside_expert_parallel_layer(P, monkeypatch):
    """Expert parallelism (peer-memory transport, one rank) routes through the
    screen: bitwise equal to the single-GPU layer."""
    from paper_2605_23911_b200.ep import ExpertParallelMoE

    monkeypatch.setenv("MOE_B200_SCREEN", "1")
    e, k, d, f, b = 64, 6, 512, 256, 96
    tokens, wr, gate, up, down = O.make_instance(31, e, k, d, f, b)
    cfg = P.ModelConfig(e, k, d, f, P.Gating("sigmoid_normalized"))
    w = P.ExpertWeights(gate, up, down)
    layer = P.MoELayer(cfg, w, wr, max_tokens=b)
    x = torch.from_numpy(tokens).cuda()
    y_ref = layer.forward(x).cpu().numpy()
    idx_ref, _ = O.route(tokens, wr, k, "sigmoid_normalized")
    bits_equal(layer.topk_idx[:b].cpu().numpy().astype(np.int64), idx_ref)
    ep = ExpertParallelMoE(cfg, wr, w, max_tokens=b, transport="p2p")
    for _ in range(2):
        bits_equal(ep.forward(x).cpu().numpy(), y_ref)
    ep.p2p.close()

