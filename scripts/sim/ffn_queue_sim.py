"""Discrete-event model of the FFN kernel's dynamic tile queue (148 SMs,
per-SM weight streaming rate, per-chunk gate+up -> down dependency) used to
choose the tile order / tail split parameters.  Usage:
  python scripts/sim/ffn_queue_sim.py"""
import heapq
import numpy as np

SMS, RATE = 148, 45e3  # bytes per us per SM (45 GB/s)
GAP = 1.2              # us of MMA idle per tile


def tiles_for(E, d, f, counts, bn, s_norm, s_tail, n_tail, lag):
    chunks = []
    for e, n in enumerate(counts):
        r = 0
        while r < n:
            chunks.append((e, min(bn, n - r)))
            r += bn
    nch = len(chunks)
    n_gu, n_dp = (f + 127) // 128, (d + 255) // 256
    gu = lambda c: [("gu", c, 2 * 128 * d * 2) for _ in range(n_gu)]
    def dn(c):
        s = s_tail if c >= nch - n_tail else s_norm
        return [("dn", c, 256 * (f // s) * 2) for _ in range(n_dp * s)]
    lag = min(lag, nch)
    order = []
    for i in range(nch):
        order += gu(i)
        if i >= lag:
            order += dn(i - lag)
    for c in range(nch - lag, nch):
        order += dn(c)
    extra = sum(n * d * 4 * 2 * ((s_tail if c >= nch - n_tail else s_norm) - 1)
                for c, (e, n) in enumerate(chunks))
    return order, nch, n_gu, extra


def simulate(order, nch, n_gu):
    free = [(0.0, i) for i in range(SMS)]
    heapq.heapify(free)
    gu_left = [n_gu] * nch
    gu_done_t = [0.0] * nch
    pending = []  # (time, chunk) completions of GU tiles
    ends = []
    t_gu_complete = {}
    gu_finish = {c: [] for c in range(nch)}
    # process in queue order: each tile goes to the earliest-free SM
    for kind, c, nbytes in order:
        t, sm = heapq.heappop(free)
        start = t
        if kind == "dn":
            start = max(t, max(gu_finish[c]))
        end = start + nbytes / RATE + GAP
        if kind == "gu":
            gu_finish[c].append(end)
        heapq.heappush(free, (end, sm))
    ts = sorted(x[0] for x in free)
    return ts[-1], np.mean(ts), ts[0]


rng = np.random.default_rng(0)
for name, E, d, f, k, B in [("mixtral", 8, 4096, 14336, 2, 512), ("qwen60", 60, 2048, 1408, 4, 512),
                            ("deepseek", 256, 7168, 2048, 8, 512), ("skew64", 64, 3584, 2560, 2, 512)]:
    counts = np.bincount(rng.integers(0, E, B * k), minlength=E)
    bn = 256 if B * k > 96 * E else 128
    base = None
    for s_norm, s_tail, n_tail, lag in [(2, 2, 0, 10**9), (2, 2, 0, 2), (2, 4, 1, 2), (2, 8, 1, 2), (2, 4, 2, 2),
                                        (2, 8, 2, 2), (2, 8, 2, 3), (1, 4, 2, 2), (1, 8, 2, 2), (2, 8, 3, 3),
                                        (1, 1, 0, 10**9), (1, 2, 4, 8), (1, 4, 8, 16), (1, 2, 16, 24)]:
        order, nch, n_gu, extra = tiles_for(E, d, f, counts, bn, s_norm, s_tail, n_tail, lag)
        mk, mean, first = simulate(order, nch, n_gu)
        extra_us = extra / 6.5e3
        print(f"{name:8s} S={s_norm} tail S={s_tail} x{n_tail} lag={lag if lag < 10**8 else 'all'}: "
              f"makespan {mk:7.1f} mean end {mean:7.1f} first {first:7.1f} +partials {extra_us:5.1f}us -> {mk + extra_us:7.1f}")
