"""Randomised shape sweep of the whole forward (GPU, through the C-ABI).

Each seed draws a layer outside the BASELINE grid -- expert counts from 1 to
512, top-k up to 32, hidden / ffn widths any multiple of 8 (ragged against
every 64-, 128- and 256-wide tile), 1 to ~700 tokens (one draw in ten
2000-5000: the streamed dispatch), either gating, fp32 or bf16 tokens,
token scales over four decades -- so the router paths (segment,
exact, INT8 screen), the chunk sizes, the down K-split counts and the combine
variants are each reached with shapes no hand-written case pins.  Routing,
counts and permutation must be bit-exact against the oracle
(oracle/moe_oracle.py: the reference's router.py / scheduler.py restated) and
y within the north_star bound of the oracle's fp32 forward on sampled tokens.
96 seeds by default (MOE_B200_FUZZ_SEEDS; 400 passed on B200 in one run).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from golden_util import bits_equal  # noqa: E402
from oracle import moe_oracle as O  # noqa: E402

TOL = 2e-2  # north_star bf16 tolerance on max|y - y_ref| / max|y_ref|
EXPERTS = (1, 2, 3, 5, 8, 16, 33, 60, 64, 128, 200, 256, 300, 512)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2605_23911_b200 as pkg
    from paper_2605_23911_b200 import _lib

    _lib.load()
    return pkg


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    e = int(rng.choice(EXPERTS))
    k = int(rng.integers(1, min(e, 32 if rng.random() < 0.2 else 8) + 1))
    d = 8 * int(rng.integers(1, 129))
    f = 8 * int(rng.integers(1, 193))
    b = int(rng.integers(1, 700)) if rng.random() < 0.9 else int(rng.integers(2000, 5000))
    b = max(1, min(b, int(3e7) // (e * d)))  # keeps the oracle's fp64 fold in memory
    gating = "softmax" if rng.random() < 0.5 else "sigmoid_normalized"
    bf16 = bool(rng.random() < 0.5)
    scale = float(10.0 ** rng.uniform(-2, 2))
    return e, k, d, f, b, gating, bf16, scale


N_SEEDS = int(os.environ.get("MOE_B200_FUZZ_SEEDS", "96"))


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_random_shape_forward(P, seed):
    e, k, d, f, b, gating, bf16, scale = _draw(seed)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((b, d), generator=gen, device="cuda") * scale
    if bf16:
        x = x.to(torch.bfloat16)
    wr = (torch.randn((d, e), generator=gen, device="cuda") / d ** 0.5).float()
    gate = (torch.randn((e * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    up = (torch.randn((e * d, f), generator=gen, device="cuda") / d ** 0.5).to(torch.bfloat16)
    down = (torch.randn((e * f, d), generator=gen, device="cuda") / f ** 0.5).to(torch.bfloat16)
    cfg = P.ModelConfig(e, k, d, f, P.Gating(gating))
    layer = P.MoELayer(cfg, P.ExpertWeights(gate, up, down), wr, max_tokens=b)
    y = layer.forward(x)
    torch.cuda.synchronize()
    assert layer.read_flags() == 0

    xf = x.float().cpu().numpy()
    wrn = wr.cpu().numpy()
    idx_ref, w_ref = O.route(xf, wrn, k, gating)
    ctx = (e, k, d, f, b, gating, bf16, scale)
    bits_equal(layer.topk_idx[:b].cpu().numpy().astype(np.int64), idx_ref)
    bits_equal(layer.topk_w[:b].cpu().numpy(), w_ref)
    bits_equal(layer.counts.cpu().numpy().astype(np.int64), O.expert_histogram(idx_ref, e))
    fwd_ref, inv_ref = O.build_permutation(idx_ref)
    bits_equal(layer.fwd[: b * k].cpu().numpy().astype(np.int64), fwd_ref)
    bits_equal(layer.inv[: b * k].cpu().numpy().astype(np.int64), inv_ref)

    def fetch(i):
        return (gate[i * d:(i + 1) * d].float().cpu().numpy(), up[i * d:(i + 1) * d].float().cpu().numpy(),
                down[i * f:(i + 1) * f].float().cpu().numpy())

    rows = np.unique(np.linspace(0, b - 1, num=min(8, b)).astype(int))
    ref = O.moe_rows(xf[rows], wrn, fetch, e, k, gating)
    err = O.max_rel_error(y.float().cpu().numpy()[rows], ref["y"])
    assert err <= TOL, (ctx, err)
