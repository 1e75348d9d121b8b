"""CPU check of the screening router's interval (csrc/router_screen.cuh).

The screen replaces each token row x and expert column w by integers
Q = rint(v 2^-u) (2^(u+19) > max|v|), splits Q into three balanced base-128
digits, accumulates the digit-plane products of weight class c = s + t
exactly (int32 on the tensor cores) and drops class 4.  It claims the
reference logit's fp64 fold (linalg.py:45-57) lies within

    V 2^(ux+uw) +- R,  V = sum_{c<=3} class_c 2^(7(4-c)),
    R = err_x S_w + err_w S_x^ + 64 min(sum|D2|, sum|G2|) 2^(ux+uw) + d u' S_x max|w|

(err = 2^(u-1), S_w = sum|w^| + d err_w >= sum|w|, S_x^ = sum|x^|,
S_x = S_x^ + d err_x).  This test restates the arithmetic in numpy / exact
rationals -- same digits, same classes, same bound -- and checks the claim
against the exact value of the sequential fp64 fold on random and adversarial
rows (huge dynamic range, subnormals, exact zeros, cancellation).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

BITS = 19


def unit_exp(vmax: float) -> int:
    if not vmax > 0:
        return 0
    _, e = np.frexp(np.float64(vmax))
    return int(e) - BITS


def digits(v: np.ndarray, ue: int):
    q = np.rint(np.ldexp(v.astype(np.float64), -ue)).astype(np.int64)
    d2 = ((q + 64) & 127) - 64
    q1 = (q - d2) >> 7
    d1 = ((q1 + 64) & 127) - 64
    d0 = (q1 - d1) >> 7
    assert np.all(np.abs(d0) <= 33) and np.all(q == d0 * 16384 + d1 * 128 + d2)
    return q, (d0, d1, d2)


def screen_interval(x: np.ndarray, w: np.ndarray):
    """(centre, radius) as exact Fractions for logit x . w (one row, one column)."""
    d = x.shape[0]
    ux, uw = unit_exp(float(np.max(np.abs(x)))), unit_exp(float(np.max(np.abs(w))))
    qx, dx = digits(x, ux)
    qw, dw = digits(w, uw)
    cls = [0, 0, 0, 0]
    for s in range(3):
        for t in range(3):
            if s + t <= 3:
                cls[s + t] += int(np.dot(dx[s], dw[t]))
    V = cls[0] * 2**28 + cls[1] * 2**21 + cls[2] * 2**14 + cls[3] * 2**7
    sc = Fraction(2) ** (ux + uw)
    err_x = Fraction(2) ** (ux - 1) if np.max(np.abs(x)) > 0 else Fraction(0)
    err_w = Fraction(2) ** (uw - 1) if np.max(np.abs(w)) > 0 else Fraction(0)
    s_xh = int(np.abs(qx).sum()) * Fraction(2) ** ux
    s_wh = int(np.abs(qw).sum()) * Fraction(2) ** uw
    s_w = s_wh + d * err_w
    s_x = s_xh + d * err_x
    drop = 64 * min(int(np.abs(dx[2]).sum()), int(np.abs(dw[2]).sum())) * sc
    gam = Fraction(d) * Fraction(2) ** -53 * Fraction(258, 256)
    wmax = Fraction(float(np.max(np.abs(w))))
    R = err_x * s_w + err_w * s_xh + drop + s_x * wmax * gam
    return V * sc, R


def fold_exact(x: np.ndarray, w: np.ndarray) -> Fraction:
    """The reference's sequential fp64 fold (np.add.accumulate of exact products)."""
    p = x.astype(np.float64) * w.astype(np.float64)
    return Fraction(float(np.add.accumulate(p)[-1]))


def _check(x, w):
    c, r = screen_interval(x, w)
    f = fold_exact(x, w)
    assert c - r <= f <= c + r, (float(c), float(r), float(f))
    return float(r)


@pytest.mark.parametrize("seed", range(8))
def test_screen_interval_random(seed):
    rng = np.random.default_rng(seed)
    d = int(rng.integers(8, 3000))
    for _ in range(20):
        x = rng.standard_normal(d).astype(np.float32)
        w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
        _check(x, w)


def test_screen_interval_adversarial():
    rng = np.random.default_rng(99)
    d = 1024
    base_w = (rng.standard_normal(d) / 32).astype(np.float32)
    cases = []
    x = rng.standard_normal(d).astype(np.float32) * np.float32(1e-6)
    x[0] = 1e3  # one huge entry: every other digit far below the row maximum
    cases.append((x, base_w))
    cases.append((np.where(rng.random(d) < 0.5, 1e-38, 3e4).astype(np.float32), base_w))  # subnormal-adjacent
    cases.append((np.zeros(d, np.float32), base_w))                                       # zero row
    x = np.full(d, 1e-40, np.float32)                                                     # subnormals only
    cases.append((x, base_w))
    x = rng.standard_normal(d).astype(np.float32)
    cases.append((x, np.float32(1e30) * base_w))                                          # huge column
    cases.append((x, np.float32(1e-30) * base_w))                                         # tiny column
    # cancellation: logit ~ 0 while sum |x w| is large
    x = np.concatenate([np.full(d // 2, 7.0), np.full(d // 2, -7.0)]).astype(np.float32)
    cases.append((x, np.abs(base_w)))
    # exactly representable values (zero quantisation error) and max-magnitude digits
    x = (rng.integers(-2**19, 2**19, d) * 2.0**-10).astype(np.float32)
    cases.append((x, (rng.integers(-2**19, 2**19, d) * 2.0**-25).astype(np.float32)))
    x = np.full(d, 2**19 - 1, np.float32)
    cases.append((x, np.full(d, -(2**19 - 1), np.float32)))
    for x, w in cases:
        _check(x, w)


def test_screen_interval_is_tight_enough_to_screen():
    """On the benched distribution (DeepSeek-V3: d = 7168, W_r ~ N(0, 1/d)),
    the radius is ~1e-3 of a unit logit: far below the gap between the k-th
    and (k+1)-th largest of 256 logits, so ~k candidates remain per token."""
    rng = np.random.default_rng(0)
    d = 7168
    x = rng.standard_normal(d).astype(np.float32)
    w = (rng.standard_normal(d) / np.sqrt(d)).astype(np.float32)
    assert _check(x, w) < 2e-3
