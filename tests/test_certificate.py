"""CPU check of the split-K logit certificate used by the segment router
(paper_2605_23911_b200/csrc/router_seg.cuh).

The reference logit is the sequential fp64 fold of exact products
(moeperf/linalg.py:45-57: np.add.accumulate).  The kernel cuts it into
segments, folds each from -0, tracks m_s = sum |partial|, merges ranges with
    C = C_l + C_r,  A = A_l + A_r + K_r |C_l|,  K = K_l + K_r
and claims the sequential value lies in [s - D, s + D], D = 2^-50 (A + |s|).
This test restates that arithmetic in numpy (same fp64 operations) and checks
the claim on random and adversarial (cancelling, wide-range, tiny) inputs.
"""

from __future__ import annotations

import numpy as np
import pytest


def _certificate(p: np.ndarray, seg_len: int, n_kb_len: int | None = None):
    """(s_hat, D) exactly as the kernel forms them (tree merges in k order)."""
    d = p.shape[0]
    nseg = (d + seg_len - 1) // seg_len
    parts = []
    for s in range(nseg):
        seg = p[s * seg_len:(s + 1) * seg_len]
        b = np.add.accumulate(np.concatenate([[-0.0], seg]))[1:]  # fold from -0
        m = 0.0
        for v in b:
            m = m + abs(v)
        parts.append((b[-1], m, float(len(seg))))

    def merge(lft, rgt):
        cl, al, kl = lft
        cr, ar, kr = rgt
        return (cl + cr, al + ar + kr * abs(cl), kl + kr)

    # pairwise tree over adjacent ranges (the kernel's shuffle tree), then sequential
    level = parts
    while len(level) > 1:
        nxt = [merge(level[i], level[i + 1]) for i in range(0, len(level) - 1, 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    s_hat, A, _ = level[0]
    D = (A + abs(s_hat)) * 2.0 ** -50
    return s_hat, A, D


def _check(x: np.ndarray, w: np.ndarray, seg_len: int):
    p = x.astype(np.float64) * w.astype(np.float64)  # exact in fp64
    seq = np.add.accumulate(p)[-1]                   # the reference fold
    s_hat, A, D = _certificate(p, seg_len)
    if A > 0:
        assert s_hat - D <= seq <= s_hat + D, (seq, s_hat, D)
        lo = np.float32(np.nextafter(s_hat - D, -np.inf))
        hi = np.float32(np.nextafter(s_hat + D, np.inf))
        assert lo <= np.float32(seq) <= hi
    return abs(seq - s_hat), D


@pytest.mark.parametrize("seg_len", [8, 16, 32, 64])
def test_certificate_random(seg_len):
    rng = np.random.default_rng(seg_len)
    worst = 0.0
    for trial in range(60):
        d = int(rng.choice([64, 512, 2048, 4096]))
        x = rng.standard_normal(d).astype(np.float32)
        w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
        err, D = _check(x, w, seg_len)
        worst = max(worst, err / D if D else 0.0)
    assert worst <= 1.0


def test_certificate_adversarial():
    rng = np.random.default_rng(7)
    cases = []
    d = 2048
    # heavy cancellation: big positive run then big negative run
    x = np.ones(d, np.float32)
    w = np.concatenate([np.full(d // 2, 1e6), np.full(d // 2, -1e6)]).astype(np.float32)
    w[::7] *= np.float32(1.0000001)
    cases.append((x, w))
    # wide dynamic range
    x = (rng.standard_normal(d) * 10.0 ** rng.integers(-30, 30, d)).astype(np.float32)
    w = (rng.standard_normal(d) * 10.0 ** rng.integers(-8, 8, d)).astype(np.float32)
    cases.append((x, w))
    # tiny values (products near the fp64 subnormal-free floor of fp32 x fp32)
    x = (rng.standard_normal(d) * 1e-38).astype(np.float32)
    w = (rng.standard_normal(d) * 1e-30).astype(np.float32)
    cases.append((x, w))
    # alternating growth: partial sums oscillate around zero
    x = np.ones(d, np.float32)
    w = ((-1.0) ** np.arange(d) * (1.0 + np.arange(d) * 1e-3)).astype(np.float32)
    cases.append((x, w))
    # bf16-valued tokens, scaled router (the throughput configs)
    x = rng.standard_normal(d).astype(np.float32)
    x = (x.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
    cases.append((x, w))
    for x, w in cases:
        for seg_len in (8, 32, 128):
            _check(x, w, seg_len)


def test_certificate_zero_is_unknown():
    """All-zero products: A == 0, the kernel marks the logit unknown (the sign of
    a zero sum depends on the order), so it is recomputed exactly."""
    p = np.zeros(64)
    p[::3] = -0.0
    _, A, _ = _certificate(p, 8)
    assert A == 0.0
