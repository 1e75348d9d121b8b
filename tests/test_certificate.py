"""CPU check of the split-K logit certificate used by the segment router
(paper_2605_23911_b200/csrc/router_seg.cuh).

The reference logit is the sequential fp64 fold of exact products
(moeperf/linalg.py:45-57: np.add.accumulate).  The kernel cuts each k-block
of kr = S*L steps into S segments of L steps, folds each from -0, tracks
m_s = sum |partial|, and merges adjacent ranges with
    C = C_l + C_r,  A = A_l + A_r + K_r |C_l|,  K = K_l + K_r
in the kernel's order: a binary shuffle tree over the 32/G segments of a warp,
then sequentially over the 8 warps, then sequentially over the k-blocks.  It
claims the sequential value lies in [s - D, s + D], D = u A (2 + 12/L)(1 + 2^-20) + 8u|s|.
This test restates that arithmetic in numpy (same fp64 operations, same
merge order) and checks the claim on random and adversarial inputs.
"""

from __future__ import annotations

import numpy as np
import pytest

U = 2.0 ** -53


def _merge(lft, rgt):
    cl, al, kl = lft
    cr, ar, kr = rgt
    return (cl + cr, al + ar + kr * abs(cl), kl + kr)


def _segment(p):
    b = np.add.accumulate(np.concatenate([[-0.0], p]))[1:]  # fold from -0
    m = 0.0
    for v in b:
        m = m + abs(v)
    return (b[-1] if len(b) else -0.0, m, float(len(p)))


def certificate(p: np.ndarray, seg_len: int, G: int = 2, threads: int = 256):
    """(s_hat, A, D) exactly as router_seg_kernel forms them."""
    d = p.shape[0]
    S = threads // G                       # segments per CTA (k-block)
    per_warp = 32 // G                     # segments per warp
    kr = S * seg_len
    total = None
    for k0 in range(0, d, kr):
        warps = []
        for w in range(S // per_warp):
            level = []
            for q in range(per_warp):
                a = k0 + (w * per_warp + q) * seg_len
                level.append(_segment(p[a:min(d, a + seg_len)] if a < d else p[:0]))
            while len(level) > 1:          # shfl_down tree: pairs of adjacent ranges
                level = [_merge(level[i], level[i + 1]) for i in range(0, len(level), 2)]
            warps.append(level[0])
        blk = (0.0, 0.0, 0.0)
        for wv in warps:                   # sequential over warps
            blk = _merge(blk, wv)
        total = blk if total is None else _merge(total, blk)  # sequential over k-blocks
    s_hat, A, _ = total
    D = A * (2.0 + 12.0 / seg_len) * (1.0 + 2.0 ** -20) * U + abs(s_hat) * 2.0 ** -50
    return s_hat, A, D


def _check(x: np.ndarray, w: np.ndarray, seg_len: int, G: int = 2):
    p = x.astype(np.float64) * w.astype(np.float64)  # exact in fp64
    seq = np.add.accumulate(p)[-1]                   # the reference fold
    s_hat, A, D = certificate(p, seg_len, G)
    if A > 0:
        assert s_hat - D <= seq <= s_hat + D, (seq, s_hat, D)
    return abs(seq - s_hat), D


@pytest.mark.parametrize("seg_len,G", [(8, 2), (16, 8), (32, 2), (32, 8), (64, 1), (128, 16)])
def test_certificate_random(seg_len, G):
    rng = np.random.default_rng(seg_len * 10 + G)
    worst = 0.0
    for _ in range(40):
        d = int(rng.choice([64, 512, 2048, 4096]))
        x = rng.standard_normal(d).astype(np.float32)
        w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
        err, D = _check(x, w, seg_len, G)
        worst = max(worst, err / D if D else 0.0)
    assert worst <= 1.0


def test_certificate_adversarial():
    rng = np.random.default_rng(7)
    d = 2048
    cases = []
    # heavy cancellation: big positive run then big negative run
    x = np.ones(d, np.float32)
    w = np.concatenate([np.full(d // 2, 1e6), np.full(d // 2, -1e6)]).astype(np.float32)
    w[::7] *= np.float32(1.0000001)
    cases.append((x, w))
    # wide dynamic range
    x = (rng.standard_normal(d) * 10.0 ** rng.integers(-30, 30, d)).astype(np.float32)
    w = (rng.standard_normal(d) * 10.0 ** rng.integers(-8, 8, d)).astype(np.float32)
    cases.append((x, w))
    # tiny values (fp32 x fp32 products stay far above the fp64 subnormal range)
    x = (rng.standard_normal(d) * 1e-38).astype(np.float32)
    w = (rng.standard_normal(d) * 1e-30).astype(np.float32)
    cases.append((x, w))
    # partial sums oscillating around zero
    x = np.ones(d, np.float32)
    w = ((-1.0) ** np.arange(d) * (1.0 + np.arange(d) * 1e-3)).astype(np.float32)
    cases.append((x, w))
    # rounding-heavy: every product a half-ulp tie relative to a large running sum
    x = np.ones(d, np.float32)
    w = np.full(d, 1.0, np.float32)
    w[0] = np.float32(2.0 ** 24)
    cases.append((x, w))
    # bf16-valued tokens, scaled router (the throughput configs)
    x = rng.standard_normal(d).astype(np.float32)
    x = (x.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
    cases.append((x, w))
    for x, w in cases:
        for seg_len, G in ((8, 2), (32, 8), (128, 1), (128, 16)):
            _check(x, w, seg_len, G)


def test_certificate_zero_is_unknown():
    """All-zero products: A == 0, the kernel marks the logit unknown (the sign of
    a zero sum depends on the order), so it is recomputed exactly."""
    p = np.zeros(64)
    p[::3] = -0.0
    _, A, _ = certificate(p, 8)
    assert A == 0.0
